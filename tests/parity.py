"""Tie-aware acceptance of GPU choices against the FP64 oracle.

Tolerances, from BASELINE.json north_star: objectives within 1e-5 relative;
where the top objectives differ by less than that, any config of the tied set
is accepted. Fairness uses an absolute band tau_f = 1e-5 around alpha (RPerf
is O(1)); DESIGN.md derives both from the FP32 arithmetic of the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np

TAU_OBJ = 1e-5
TAU_F = 1e-5

# Conditioning (reading R25): the CUDA path evaluates each RPerf and
# each objective as short FP32 sums of the model's terms C_t*H_t and D_t*J_t
# (P:L458); its rounding error is at most ~KAPPA unit roundoffs of the SUM OF
# THE TERMS' MAGNITUDES M, not of the result. When the terms cancel (an RPerf
# or a Throughput near 0, e.g. alpha = 0 with tiny objectives) no FP32
# evaluation resolves 1e-5 relative, so each band is max(tau * |value|,
# KAPPA * u32 * M): tau wherever the value is not cancellation-dominated.
U32 = 2.0 ** -24
KAPPA = 16


def _coefs(pb):
    C = np.asarray(pb.coef_c, np.float64)
    D = np.asarray(pb.coef_d, np.float64)
    caps = np.asarray(pb.caps_w, np.float32)
    invp = 1.0 / caps.astype(np.float64) if pb.objective == 2 else np.ones(len(caps))
    return C, D, invp


def term_magnitudes(pb, rows):
    """Per config c = state * n_caps + cap of the set `rows`: (M_obj[c], M_fair[c]) with
    M_obj = sum over slots of the |terms| entering Throughput (/P), M_fair = max over
    slots of |alpha| + the |terms| of that slot's RPerf."""
    import oracle
    C, D, invp = _coefs(pb)
    ns = len(rows)
    MU = np.stack([np.abs(C * oracle.basis_h(f)).sum(-1) for f in rows])  # [slot][cap][slice]
    MV = np.stack([np.abs(D * oracle.basis_j(f)).sum(-1) for f in rows])
    sl = np.asarray(pb.state_slice)  # [state][slot]
    per_slot = []
    for i in range(ns):
        m = MU[i][:, sl[:, i]]  # [cap][state]
        for l in range(ns):
            if l != i:
                m = m + MV[l][:, sl[:, i]]
        per_slot.append(m.T)  # [state][cap]
    per_slot = np.stack(per_slot)
    mobj = (per_slot.sum(0) * invp[None, :]).reshape(-1)
    mfair = (per_slot.max(0) + abs(float(np.float32(pb.alpha)))).reshape(-1)
    return mobj, mfair


def chosen_obj_magnitudes(pb, F, cfg, jobs=None):
    """M_obj of every set of the queue (colex order) at its config cfg[k] (>= 0); 0 where cfg < 0.
    Vectorised form of term_magnitudes for the full-queue objective check."""
    import oracle
    C, D, invp = _coefs(pb)
    rows = F if jobs is None else F[np.asarray(jobs)]
    H = np.stack([oracle.basis_h(f) for f in rows])
    J = np.stack([oracle.basis_j(f) for f in rows])
    MU = np.einsum("pst,nt->nsp", np.abs(C), np.abs(H))  # sum_t |C_t H_t| per job, slice, cap
    MV = np.einsum("pst,nt->nsp", np.abs(D), np.abs(J))
    n, ns = rows.shape[0], pb.n_slots
    ncap = len(invp)
    if ns == 2:
        j1 = np.repeat(np.arange(n), np.arange(n))
        j0 = np.concatenate([np.arange(k) for k in range(n)])
        pos = [j0, j1]
    else:
        trip = [(a, b, c) for c in range(n) for b in range(c) for a in range(b)]
        pos = [np.array([t[i] for t in trip], dtype=np.int64) for i in range(3)]
    cfg = np.asarray(cfg)
    ok = cfg >= 0
    c = np.where(ok, cfg, 0)
    st, p = c // ncap, c % ncap
    m = np.zeros(len(cfg))
    for i in range(ns):
        sl = pb.state_slice[st, i]
        m += MU[pos[i], sl, p]
        for l in range(ns):
            if l != i:
                m += MV[pos[l], sl, p]
    return np.where(ok, m * invp[p], 0.0)


def obj_band(obj_o, mobj, tau_obj=TAU_OBJ):
    return np.maximum(tau_obj * np.abs(obj_o), KAPPA * U32 * np.asarray(mobj)) + 1e-12


def accept_set(obj_o, fair_o, alpha, cfg_g, obj_g, tau_obj=TAU_OBJ, tau_f=TAU_F, mobj=None, mfair=None):
    """(ok, reason) for one set: obj_o/fair_o are the oracle's per-config values (FP64);
    mobj/mfair the per-config term magnitudes (term_magnitudes; None = well conditioned)."""
    n = len(obj_o)
    mobj = np.zeros(n) if mobj is None else np.asarray(mobj)
    mfair = np.zeros(n) if mfair is None else np.asarray(mfair)
    band_f = np.maximum(tau_f, KAPPA * U32 * mfair)
    strict = fair_o > alpha + band_f
    loose = fair_o > alpha - band_f
    if cfg_g < 0:
        return (not strict.any(), "gpu says infeasible but a config is strictly feasible")
    if not loose[cfg_g]:
        return False, f"cfg {cfg_g} is infeasible (fair {fair_o[cfg_g]!r} <= alpha {alpha})"
    o = obj_o[cfg_g]
    if abs(obj_g - o) > obj_band(o, mobj[cfg_g], tau_obj):
        return False, f"obj {obj_g!r} vs oracle {o!r} at cfg {cfg_g}"
    if strict.any():
        # the chosen config's objective may sit below the strict best by tau (the tie
        # rule) plus what FP32 rounding can move either of them (the conditioning bands)
        lo_best = (obj_o - KAPPA * U32 * mobj)[strict].max()
        best = obj_o[strict].max()
        if o + KAPPA * U32 * mobj[cfg_g] < lo_best - tau_obj * abs(best):
            return False, f"cfg {cfg_g} obj {o!r} < strict best {best!r}"
    return True, ""


def check_sets(orc, F, jobs, set_ids, cfg_g, obj_g, n_jobs, n_slots):
    """Check GPU (cfg, obj) for the listed set ids; returns (n_exact_index, failures)."""
    import oracle
    fails = []
    exact = 0
    for sid, c, o in zip(set_ids, cfg_g, obj_g):
        pos = oracle.unrank(n_jobs, n_slots, int(sid))
        rows = [F[jobs[p]] if jobs is not None else F[p] for p in pos]
        obj_o, fair_o, thr_o, feas_o, rp_o = orc.eval_set(rows)
        c_o, _ = orc.best_config(rows)
        exact += int(c_o == int(c))
        mobj, mfair = term_magnitudes(orc.pb, rows)
        ok, why = accept_set(obj_o, fair_o, float(np.float32(orc.pb.alpha)), int(c), float(o), mobj=mobj,
                             mfair=mfair)
        if not ok:
            fails.append((int(sid), why))
    return exact, fails


def replay_greedy(n_jobs, n_slots, set_obj_oracle, picks, tau_obj=TAU_OBJ):
    """Tie-aware replay of a greedy pick list: pick t must be disjoint from the earlier picks,
    feasible, and within tau_obj of the oracle's best remaining disjoint set."""
    import oracle
    order = np.lexsort((np.arange(len(set_obj_oracle)), -set_obj_oracle))
    feasible = set_obj_oracle > -math.inf
    taken = np.zeros(n_jobs, dtype=bool)
    members = {}

    def mem(sid):
        if sid not in members:
            members[sid] = oracle.unrank(n_jobs, n_slots, int(sid))
        return members[sid]

    ptr = 0
    for t, g in enumerate(picks):
        while ptr < len(order) and (not feasible[order[ptr]] or taken[list(mem(order[ptr]))].any()):
            ptr += 1
        if ptr >= len(order):
            return False, f"pick {t}: oracle has no remaining set"
        best = set_obj_oracle[order[ptr]]
        if not feasible[g] or taken[list(mem(g))].any():
            return False, f"pick {t}: set {g} infeasible or overlaps"
        if set_obj_oracle[g] < best - tau_obj * abs(best):
            return False, f"pick {t}: set {g} obj {set_obj_oracle[g]!r} < best remaining {best!r}"
        taken[list(mem(g))] = True
    return True, ""

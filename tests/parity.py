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


def accept_set(obj_o, fair_o, alpha, cfg_g, obj_g, tau_obj=TAU_OBJ, tau_f=TAU_F):
    """(ok, reason) for one set: obj_o/fair_o are the oracle's per-config values (FP64)."""
    strict = fair_o > alpha + tau_f
    loose = fair_o > alpha - tau_f
    if cfg_g < 0:
        return (not strict.any(), "gpu says infeasible but a config is strictly feasible")
    if not loose[cfg_g]:
        return False, f"cfg {cfg_g} is infeasible (fair {fair_o[cfg_g]!r} <= alpha {alpha})"
    o = obj_o[cfg_g]
    if abs(obj_g - o) > tau_obj * abs(o) + 1e-12:
        return False, f"obj {obj_g!r} vs oracle {o!r} at cfg {cfg_g}"
    if strict.any():
        best = obj_o[strict].max()
        if o < best - tau_obj * abs(best):
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
        ok, why = accept_set(obj_o, fair_o, float(np.float32(orc.pb.alpha)), int(c), float(o))
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

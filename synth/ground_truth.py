"""A synthetic GPU standing in for the paper's measurement campaign (SPEC.md
module `oracle`, L430-470; §5.1.3: "execute these benchmarks
with exclusive solo-runs while scaling the power and hardware resource
allocations ... measure performance degradation", then co-runs).

This is INPUT construction for the calibration step:
it produces "measured" relative performances for training samples. It is not
the paper's model (no basis function, no C/D coefficients): it is SPEC's
roofline-style simulator of compute supply under a power cap and memory supply
under the shared/private options, so a linear fit of the paper's model to it
is a genuine regression, not an identity.

Per SPEC `true_rperf` (a)-(f): for the apps co-located on a state (gpcs g_i,
memory option) under cap P
  c_eff_i   = c_i (1 + kappa t_i)
  draw      = w_base + w_gpc sum_i g_i c_eff_i
  throttle  = clamp((P - w_base) / (draw - w_base), f_min, 1) if draw > P else 1
  compute_i = (g_i / G_full) throttle
  memory_i  = m(g_i) / modules (private) | b_i or b_i / sum b (shared, demand-proportional)
  rperf_i   = min(1, compute_i / c_i, memory_i / b_i)   (b term dropped when b_i = 0)
divided by the same expression for the app alone on the full chip at P_max.
App parameters come from the counter vector (SPEC `synthesize_profile`
inverted): c = F1/100, b = F3/100, t = (F6+F7+F8)/F1.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Tuple

import numpy as np

from .generator import G_FULL, Problem, SplitMix64


@dataclass(frozen=True)
class GPUModel:
    g_full: int
    modules: Dict[int, int]  # private option: GPCs -> memory modules
    n_modules: int
    w_base: float
    w_gpc: float
    kappa: float
    f_min: float
    p_max: float


# SPEC.md defaults (A100: 1,2,4,4,8 modules for 1,2,3,4,7 GPCs, §3) and a
# B200-like variant (8 GPCs, one module per GPC, 500-1000 W caps). Simulation
# parameters, not hardware claims.
A100 = GPUModel(8, {1: 1, 2: 2, 3: 4, 4: 4, 7: 8, 8: 8}, 8, 50.0, 25.0, 0.6, 0.1, 250.0)
B200 = GPUModel(8, {g: g for g in range(1, 9)}, 8, 200.0, 110.0, 0.6, 0.1, 1000.0)


def app_params(F: np.ndarray) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    F = np.asarray(F, dtype=np.float64)
    c = F[:, 0] / 100.0
    b = F[:, 2] / 100.0
    t = np.where(F[:, 0] > 0, (F[:, 5] + F[:, 6] + F[:, 7]) / np.maximum(F[:, 0], 1e-12), 0.0)
    return c, b, t


def _raw(model: GPUModel, c, b, t, gpcs, mem: int, P: float) -> np.ndarray:
    """Un-normalised rperf of every co-located app (arrays over slots, broadcast over samples)."""
    c_eff = [ci * (1.0 + model.kappa * ti) for ci, ti in zip(c, t)]
    draw = model.w_base + model.w_gpc * sum(g * ce for g, ce in zip(gpcs, c_eff))
    thr = np.where(draw > P, np.clip((P - model.w_base) / np.maximum(draw - model.w_base, 1e-12), model.f_min, 1.0),
                   1.0)
    bsum = sum(b)
    out = []
    for i, g in enumerate(gpcs):
        comp = (g / model.g_full) * thr
        if mem == 1:
            memory = model.modules[g] / model.n_modules
        else:
            memory = np.where(bsum <= 1.0, b[i], b[i] / np.maximum(bsum, 1e-12))
        r = np.minimum(1.0, comp / c[i])
        r = np.where(b[i] > 0, np.minimum(r, memory / np.maximum(b[i], 1e-12)), r)
        out.append(r)
    return np.stack(out)


def true_rperf(model: GPUModel, F_slots, gpcs, mem: int, P: float) -> np.ndarray:
    """[n_slots][n] true relative performance of each slot's app (F_slots: per-slot [n][8])."""
    params = [app_params(F) for F in F_slots]
    c = [p[0] for p in params]
    b = [p[1] for p in params]
    t = [p[2] for p in params]
    raw = _raw(model, c, b, t, gpcs, mem, P)
    base = np.stack([_raw(model, [c[i]], [b[i]], [t[i]], (model.g_full,), 0, model.p_max)[0]
                     for i in range(len(gpcs))])
    return raw / base


@dataclass
class TrainingSet:
    """Calibration samples; key = cap * n_slices + slice (the row of coef_c / coef_d)."""
    n_slices: int
    n_caps: int
    n_slots: int
    solo_app: np.ndarray = field(default=None)       # int32 [n_solo]
    solo_key: np.ndarray = field(default=None)       # int32 [n_solo]
    solo_rperf: np.ndarray = field(default=None)     # float32 [n_solo]
    co_app: np.ndarray = field(default=None)         # int32 [n_co]
    co_partners: np.ndarray = field(default=None)    # int32 [n_co][n_slots - 1]
    co_key: np.ndarray = field(default=None)         # int32 [n_co]
    co_rperf: np.ndarray = field(default=None)       # float32 [n_co]


def _gauss(rng: SplitMix64, n: int) -> np.ndarray:
    u1 = np.maximum(rng.uniform(n), 1e-300)
    u2 = rng.uniform(n)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def make_training_set(F: np.ndarray, pb: Problem, n_corun: int, seed: int, noise: float = 0.0,
                      model: GPUModel = B200, solo_apps: int | None = None) -> TrainingSet:
    """Solo samples of the first `solo_apps` apps (default all) on every slice x cap,
    and `n_corun` random co-runs (distinct apps, random state and cap, one sample per
    slot), measured on the synthetic GPU, plus optional Gaussian noise (SPEC default 0)."""
    F = np.asarray(F, dtype=np.float32)
    n = F.shape[0]
    ns, nsl, nc = pb.n_slots, pb.n_slices, pb.n_caps
    rng = SplitMix64(seed)
    na = n if solo_apps is None else min(n, solo_apps)
    # solo: every (app, slice, cap)
    apps, keys, ys = [], [], []
    for s, (g, m) in enumerate(pb.slices):
        for p in range(nc):
            y = true_rperf(model, [F[:na]], (g,), m, float(pb.caps_w[p]))[0]
            apps.append(np.arange(na, dtype=np.int32))
            keys.append(np.full(na, p * nsl + s, dtype=np.int32))
            ys.append(y)
    solo_app = np.concatenate(apps)
    solo_key = np.concatenate(keys)
    solo_y = np.concatenate(ys)
    # co-runs: random distinct apps, state, cap
    co_app = co_key = co_y = None
    co_part = np.zeros((0, max(ns - 1, 0)), dtype=np.int32)
    if n_corun > 0 and ns > 1:
        sel = np.zeros((n_corun, ns), dtype=np.int64)
        for i in range(ns):
            sel[:, i] = (rng.uniform(n_corun) * n).astype(np.int64) % n
        for i in range(1, ns):  # make the apps of a co-run distinct
            for j in range(i):
                clash = sel[:, i] == sel[:, j]
                sel[clash, i] = (sel[clash, i] + 1 + j) % n
        st = (rng.uniform(n_corun) * pb.n_states).astype(np.int64) % pb.n_states
        cp = (rng.uniform(n_corun) * nc).astype(np.int64) % nc
        a_l, p_l, k_l, y_l = [], [], [], []
        for s in range(pb.n_states):
            for p in range(nc):
                idx = np.nonzero((st == s) & (cp == p))[0]
                if idx.size == 0:
                    continue
                gp = tuple(int(x) for x in pb.state_gpcs[s])
                y = true_rperf(model, [F[sel[idx, i]] for i in range(ns)], gp, int(pb.state_mem[s]),
                               float(pb.caps_w[p]))
                for i in range(ns):
                    a_l.append(sel[idx, i])
                    p_l.append(np.stack([sel[idx, l] for l in range(ns) if l != i], axis=1))
                    k_l.append(np.full(idx.size, p * nsl + int(pb.state_slice[s, i]), dtype=np.int64))
                    y_l.append(y[i])
        co_app = np.concatenate(a_l).astype(np.int32)
        co_part = np.concatenate(p_l).astype(np.int32)
        co_key = np.concatenate(k_l).astype(np.int32)
        co_y = np.concatenate(y_l)
    if noise > 0:
        solo_y = solo_y + noise * _gauss(rng, solo_y.size)
        if co_y is not None:
            co_y = co_y + noise * _gauss(rng, co_y.size)
    ts = TrainingSet(n_slices=nsl, n_caps=nc, n_slots=ns, solo_app=solo_app, solo_key=solo_key,
                     solo_rperf=solo_y.astype(np.float32))
    if co_y is not None:
        ts.co_app, ts.co_partners, ts.co_key, ts.co_rperf = co_app, co_part, co_key, co_y.astype(np.float32)
    else:
        ts.co_app = np.zeros(0, np.int32)
        ts.co_partners = co_part
        ts.co_key = np.zeros(0, np.int32)
        ts.co_rperf = np.zeros(0, np.float32)
    return ts

"""CPU oracle of the worst / proposal / best evaluation
-- TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's cpu_baseline leg).

PAPER.md §5.2.2: "The worst/best chooses one partitioning/allocation state
(S) from those meet the fairness constraint"; L777: the geometric means of the
worst, the proposal and the best. For every set: the proposal (the search's
config) is scored by the ground truth; best / worst are the largest / smallest
ground-truth objective (Throughput, or Throughput / P for Problem 2) over the
configs whose ground-truth Fairness (min RPerf) exceeds alpha. The ground truth
is the synthetic GPU of synth/ground_truth.py (SPEC.md true_rperf; reading R21),
evaluated here in FP64 straight from its definition.
"""
from __future__ import annotations

import math

import numpy as np

from . import n_sets, unrank
from synth.ground_truth import true_rperf


def set_members(n_jobs: int, n_slots: int, first: int, count: int) -> np.ndarray:
    """[count][n_slots] ascending queue positions of sets first .. first+count-1."""
    return np.array([unrank(n_jobs, n_slots, s) for s in range(first, first + count)], dtype=np.int64).reshape(
        count, n_slots)


def worst_prop_best(pb, F, prop_cfg, model, jobs=None, first: int = 0, count=None):
    """(prop_obj, prop_fair, best_obj, worst_obj) per set, FP64."""
    F = np.asarray(F, dtype=np.float32)
    n_jobs = F.shape[0] if jobs is None else len(jobs)
    if count is None:
        count = n_sets(n_jobs, pb.n_slots) - first
    mem = set_members(n_jobs, pb.n_slots, first, count)
    rows = mem if jobs is None else np.asarray(jobs)[mem]
    Fs = [F[rows[:, i]] for i in range(pb.n_slots)]
    nc = pb.n_caps
    prop_cfg = np.asarray(prop_cfg)
    best = np.full(count, -math.inf)
    worst = np.full(count, math.inf)
    p_obj = np.full(count, -math.inf)
    p_fair = np.full(count, -math.inf)
    alpha = float(np.float32(pb.alpha))
    for s in range(pb.n_states):
        gp = tuple(int(g) for g in pb.state_gpcs[s])
        for p in range(nc):
            P = float(pb.caps_w[p])
            r = true_rperf(model, Fs, gp, int(pb.state_mem[s]), P)  # [n_slots][count]
            thr = r.sum(axis=0)
            fair = r.min(axis=0)
            obj = thr / P if pb.objective == 2 else thr
            ok = fair > alpha
            best = np.where(ok, np.maximum(best, obj), best)
            worst = np.where(ok, np.minimum(worst, obj), worst)
            hit = prop_cfg == s * nc + p
            p_obj = np.where(hit, obj, p_obj)
            p_fair = np.where(hit, fair, p_fair)
    worst = np.where(best > -math.inf, worst, -math.inf)
    return p_obj, p_fair, best, worst


def summary(pb, prop_cfg, p_obj, p_fair, best, worst):
    """Geometric means over the sets with a proposal and a truly feasible config."""
    m = (np.asarray(prop_cfg) >= 0) & (best > -math.inf)
    n = int(m.sum())
    alpha = float(np.float32(pb.alpha))
    return {"n_compared": n, "n_violations": int((p_fair[m] <= alpha).sum()),
            "geomean_prop_over_best": float(np.exp(np.mean(np.log(p_obj[m] / best[m])))) if n else math.nan,
            "geomean_worst_over_best": float(np.exp(np.mean(np.log(worst[m] / best[m])))) if n else math.nan}

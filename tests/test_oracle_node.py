"""Pins of the node power-budget oracle (NEXT #4; oracle/node_budget.py, reading R23)
against brute force and the special cases that reduce to the per-set search. CPU only."""
import math

import numpy as np
import pytest

from oracle import Oracle, unrank
from oracle import node_budget as nb
from synth import make_features, make_problem


def _fronts(o, F, sets, n_jobs):
    return [nb.frontier(o, [F[p] for p in unrank(n_jobs, o.pb.n_slots, s)]) for s in sets]


@pytest.mark.parametrize("objective", [1, 2])
def test_dp_equals_brute_force(objective):
    pb = make_problem("a100_paper", "a100_paper", coef_seed=3, alpha=0.2, objective=objective)
    F, _ = make_features(12, seed=3)
    o = Oracle(pb)
    sets = [0, 13, 40]
    fr = [f for f, _ in _fronts(o, F, sets, 12)]
    for node_w in (450.0, 560.0, 640.0, 750.0, 1000.0):
        v, caps = nb.solve_node(fr, pb.caps_w, node_w, objective)
        bv, bcaps = nb.brute_node(fr, pb.caps_w, node_w, objective)
        assert (v == bv == -math.inf) or abs(v - bv) <= 1e-12 * abs(bv)
        if caps:
            assert sum(float(pb.caps_w[p]) for p in caps) <= node_w
            t = sum(f[p] for f, p in zip(fr, caps))
            assert abs((t if objective == 1 else t / sum(float(pb.caps_w[p]) for p in caps)) - v) <= 1e-12


def test_single_gpu_unlimited_budget_is_the_per_set_search():
    """One GPU with a budget of its largest cap (no constraint): Problem 2's node optimum is the set's exhaustive
    Throughput/P optimum and Problem 1's is its best feasible Throughput."""
    pb2 = make_problem("b200", "c21", coef_seed=4, alpha=0.3, objective=2)
    F, _ = make_features(20, seed=4)
    o2 = Oracle(pb2)
    for s in (0, 77, 150):
        rows = [F[p] for p in unrank(20, 2, s)]
        f, st = nb.frontier(o2, rows)
        v, caps = nb.solve_node([f], pb2.caps_w, 1000.0, 2)
        c, obj = o2.best_config(rows)
        if c < 0:
            assert v == -math.inf
        else:
            assert abs(v - obj) <= 1e-12 * abs(obj)
            assert caps == [c % pb2.n_caps] and st[caps[0]] == c // pb2.n_caps
    pb1 = make_problem("b200", "c21", coef_seed=4, alpha=0.3, objective=1)
    o1 = Oracle(pb1)
    rows = [F[0], F[5]]
    _, _, thr, feas, _ = o1.eval_set(rows)
    f, _ = nb.frontier(o1, rows)
    v, caps = nb.solve_node([f], pb1.caps_w, 1000.0, 1)
    assert v == (thr[feas].max() if feas.any() else -math.inf)


def test_budget_monotone_and_infeasible():
    pb = make_problem("b200", "c10", coef_seed=5, alpha=0.2, objective=1)
    F, _ = make_features(30, seed=5)
    o = Oracle(pb)
    fr = [f for f, _ in _fronts(o, F, [3, 100, 200, 300], 30)]
    prev = -math.inf
    for node_w in range(2200, 4200, 100):
        v, _ = nb.solve_node(fr, pb.caps_w, float(node_w), 1)
        assert v >= prev
        prev = v
    assert nb.solve_node(fr, pb.caps_w, 2100.0, 1)[0] == -math.inf  # 4 x 550 W minimum

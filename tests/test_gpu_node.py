"""GPU node-level power budgeting (cosched_node_budget, NEXT #4) vs the FP64 DP oracle
(oracle/node_budget.py, reading R23).

Bar: per node, the GPU's choice respects the budget, puts every GPU on a config the
oracle finds feasible (up to tau_f), and its objective -- re-evaluated by the oracle --
is within 1e-5 relative of the oracle's optimum; the reported node objective matches
the oracle's value of the GPU's choice within 1e-5.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import Oracle, unrank  # noqa: E402
from oracle import node_budget as nb  # noqa: E402
from synth import bench_config, make_features, make_problem  # noqa: E402
from parity import TAU_F, TAU_OBJ  # noqa: E402


@pytest.fixture(scope="module")
def cs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03838_b200 as cs
    return cs


def _check(cs, pb, F, sets, G, node_w):
    s = cs.Scheduler(pb)
    s.score_all(torch.from_numpy(F).cuda())
    caps, cfgs, nobj = s.node_budget(sets, G, node_w, pb.objective)
    o = Oracle(pb)
    n = F.shape[0]
    alpha = float(np.float32(pb.alpha))
    for k in range(len(sets) // G):
        grp = sets[k * G:(k + 1) * G]
        rows = [[F[p] for p in unrank(n, pb.n_slots, sid)] for sid in grp]
        fr = [nb.frontier(o, r)[0] for r in rows]
        ov, ocaps = nb.solve_node(fr, pb.caps_w, node_w, pb.objective)
        gc = caps[k * G:(k + 1) * G]
        if ov == -math.inf:
            assert nobj[k] == -math.inf and all(c == -1 for c in gc)
            continue
        assert all(c >= 0 for c in gc)
        P = sum(float(pb.caps_w[c]) for c in gc)
        assert P <= node_w
        tot = 0.0
        for r, cfg in zip(rows, cfgs[k * G:(k + 1) * G]):
            _, fair, thr, _, _ = o.eval_set(r)
            assert fair[cfg] > alpha - TAU_F
            tot += thr[cfg]
        val = tot if pb.objective == 1 else tot / P
        assert val >= ov * (1 - TAU_OBJ), (k, val, ov)
        assert abs(nobj[k] - val) <= TAU_OBJ * abs(val)
    return caps, cfgs, nobj


@pytest.mark.parametrize("objective", [1, 2])
def test_node_budget_pairs(cs, objective):
    pb = make_problem("b200", "c21", coef_seed=111, alpha=0.25, objective=objective)
    F, _ = make_features(64, seed=112)
    rng = np.random.default_rng(113)
    sets = [int(x) for x in rng.integers(0, 64 * 63 // 2, 8 * 6)]
    for node_w in (4500.0, 5600.0, 8000.0):
        _check(cs, pb, F, sets, 8, node_w)


def test_node_budget_triples_and_a100(cs):
    pb = make_problem("b200_3way", "c10", coef_seed=114, alpha=0.2, objective=2)
    F, _ = make_features(30, seed=115)
    _check(cs, pb, F, [0, 100, 2000, 3000], 4, 3000.0)
    pb = make_problem("a100_paper", "a100_paper", coef_seed=116, alpha=0.2, objective=1)
    F, _ = make_features(20, seed=117)
    _check(cs, pb, F, [0, 5, 17, 44, 90, 120], 3, 600.0)


def test_allocation_then_budget_at_c4_scale(cs):
    """The job manager's pipeline: greedy allocation of C4 onto 5,000 GPUs, then caps for
    625 nodes of 8 GPUs under a 6 kW budget; sampled nodes match the oracle."""
    pb, F = bench_config("C4")
    s = cs.Scheduler(pb)
    s.score_all(torch.from_numpy(F).cuda())
    st, ids, _, _ = s.best_allocation(5000)
    assert st == 0 and len(ids) == 5000
    caps, cfgs, nobj = s.node_budget(ids, 8, 6000.0, 2)
    assert len(nobj) == 625 and all(v > 0 for v in nobj)
    o = Oracle(pb)
    for k in (0, 311, 624):
        grp = ids[k * 8:(k + 1) * 8]
        fr = [nb.frontier(o, [F[p] for p in unrank(10000, 2, sid)])[0] for sid in grp]
        ov, _ = nb.solve_node(fr, pb.caps_w, 6000.0, 2)
        assert abs(nobj[k] - ov) <= 1e-5 * abs(ov)
        assert sum(float(pb.caps_w[c]) for c in caps[k * 8:(k + 1) * 8]) <= 6000.0


def test_errors(cs):
    pb = make_problem("b200", "c10", coef_seed=118)
    F, _ = make_features(10, seed=118)
    s = cs.Scheduler(pb)
    with pytest.raises(cs.CoschedError):
        s.node_budget([0, 1], 2, 2000.0, 2)  # before score_all
    s.score_all(torch.from_numpy(F).cuda())
    with pytest.raises(cs.CoschedError):
        s.node_budget([0, 1, 2], 2, 2000.0, 2)  # not a multiple of gpus_per_node
    with pytest.raises(cs.CoschedError):
        s.node_budget([0, 1000], 2, 2000.0, 2)  # set id out of range
    with pytest.raises(cs.CoschedError):
        s.node_budget([0, 1], 2, 1e9, 2)  # too many budget units

"""Pins of the worst / proposal / best oracle (NEXT #3; oracle/evaluate.py) against
brute force and the cases SPEC.md compare_worst_best fixes. CPU only."""
import math

import numpy as np

from oracle import Oracle, unrank
from oracle import evaluate as ev
from synth import make_features, make_problem
from synth.ground_truth import A100, B200, true_rperf


def test_brute_force_extremes_and_proposal():
    """best / worst are the extremes of the truth objective over truly feasible configs
    and the proposal is the truth at the given config (checked config by config)."""
    pb = make_problem("b200", "c10", coef_seed=3, alpha=0.25)
    F, _ = make_features(12, seed=3)
    n_sets = 66
    prop = np.arange(n_sets) % pb.n_configs
    po, pf, best, worst = ev.worst_prop_best(pb, F, prop, B200)
    for sid in (0, 17, 65):
        rows = [F[p] for p in unrank(12, 2, sid)]
        vals, fairs = [], []
        for s in range(pb.n_states):
            for p in range(pb.n_caps):
                r = true_rperf(B200, [r_[None] for r_ in rows], tuple(pb.state_gpcs[s]), int(pb.state_mem[s]),
                               float(pb.caps_w[p]))[:, 0]
                vals.append(r.sum() / float(pb.caps_w[p]))
                fairs.append(r.min())
        vals, fairs = np.array(vals), np.array(fairs)
        ok = fairs > np.float32(0.25)
        assert best[sid] == (vals[ok].max() if ok.any() else -math.inf)
        assert worst[sid] == (vals[ok].min() if ok.any() else -math.inf)
        assert po[sid] == vals[prop[sid]] and pf[sid] == fairs[prop[sid]]
        assert worst[sid] <= best[sid]


def test_single_config_space_gives_ratio_one():
    """With one state and one cap, proposal = best = worst: every ratio is 1 (SPEC: proposal =
    best on a dominance landscape -> ratio 1.0)."""
    pb = make_problem("b200", "c1_1000", coef_seed=4, alpha=0.0, objective=1)
    pb.state_gpcs, pb.state_mem, pb.state_slice = pb.state_gpcs[:1], pb.state_mem[:1], pb.state_slice[:1]
    F, _ = make_features(10, seed=4)
    po, pf, best, worst = ev.worst_prop_best(pb, F, np.zeros(45, dtype=np.int64), B200)
    sm = ev.summary(pb, np.zeros(45), po, pf, best, worst)
    assert sm["n_compared"] == 45 and sm["geomean_prop_over_best"] == 1.0 and sm["geomean_worst_over_best"] == 1.0


def test_misranking_table_shows_the_gap():
    """A proposal that is not the truth argmax reports proposal / best < 1 (SPEC adversarial
    example); the model's own choice on a fitted table is closer to the best than the worst."""
    pb = make_problem("a100_paper", "a100_paper", coef_seed=5, alpha=0.2, objective=1)
    F, _ = make_features(8, seed=5)
    fixed = np.zeros(28, dtype=np.int64)  # always S1 at 150 W: misranks most sets
    po, pf, best, worst = ev.worst_prop_best(pb, F, fixed, A100)
    m = best > -math.inf
    sm0 = ev.summary(pb, fixed, po, pf, best, worst)
    assert sm0["geomean_prop_over_best"] < 0.99  # the gap is reported
    o = Oracle(pb)
    prop = np.array([o.best_config([F[p] for p in unrank(8, 2, s)])[0] for s in range(28)])
    po2, pf2, _, _ = ev.worst_prop_best(pb, F, prop, A100)
    sm = ev.summary(pb, prop, po2, pf2, best, worst)
    assert sm["geomean_worst_over_best"] <= sm["geomean_prop_over_best"] <= 1.0 + 1e-12
    assert sm["geomean_prop_over_best"] > sm0["geomean_prop_over_best"]

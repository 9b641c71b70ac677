"""Pins of the oracle's hill climb (NEXT #2; P:L664 / L796; reading R22)
against brute force and the properties SPEC.md L352-377 fixes. CPU only."""
import math

import numpy as np

from oracle import Oracle
from synth import make_features, make_problem


def test_hill_climb_never_beats_exhaustive_and_is_a_local_optimum():
    """obj(hill) <= obj(exhaustive) on every input, and the result is a
    local optimum of the feasibility-filtered landscape (checked by brute force)."""
    pb = make_problem("b200", "c10", coef_seed=5, alpha=0.3)
    F, _ = make_features(30, seed=5)
    o = Oracle(pb)
    ns, nc = pb.n_states, pb.n_caps
    for a in range(0, 30, 3):
        for b in range(a + 1, 30, 4):
            rows = [F[a], F[b]]
            objs, fair, _, feas, _ = o.eval_set(rows)
            f = np.where(feas, objs, -np.inf).reshape(ns, nc)
            c_ex, o_ex = o.best_config(rows)
            for start in ((0, 0), (ns - 1, nc - 1), (3, 5)):
                c, v, ev = o.hill_climb(rows, *start)
                assert v <= o_ex
                if c < 0:
                    assert c_ex < 0
                    continue
                s, p = divmod(c, nc)
                assert f[s, p] == v
                for ds, dp in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                    if 0 <= s + ds < ns and 0 <= p + dp < nc:
                        assert not (f[s + ds, p + dp] > v)


def test_unimodal_landscape_matches_exhaustive_and_optimum_start_is_fixed_point():
    """On a unimodal landscape (constant-only C peaked at one (state, cap), D = 0) the climb
    from any start reaches the exhaustive optimum; starting at the optimum it
    stays after evaluating itself and its neighbours."""
    pb = make_problem("b200", "c10", coef_seed=6, alpha=0.0, objective=1)
    ns, nc = pb.n_states, pb.n_caps
    s_pk, p_pk = 4, 6
    # RPerf = 1 - 0.05 (|s - s_pk| + |p - p_pk|) on both slots; each state gets its own
    # pair of coefficient rows (full-state keying, reading R1)
    ss = np.arange(ns * 2, dtype=np.int32).reshape(ns, 2)
    C = np.zeros((nc, ns * 2, 6), dtype=np.float32)
    for s in range(ns):
        for p in range(nc):
            C[p, ss[s], 5] = 1 - 0.05 * (abs(s - s_pk) + abs(p - p_pk))
    pb.state_slice = ss
    pb.slices = [(0, 0)] * (ns * 2)
    pb.coef_c = C
    pb.coef_d = np.zeros((nc, ns * 2, 3), dtype=np.float32)
    o = Oracle(pb)
    F, _ = make_features(4, seed=6)
    rows = [F[0], F[1]]
    c_ex, o_ex = o.best_config(rows)
    assert c_ex == s_pk * nc + p_pk
    for start in ((0, 0), (ns - 1, 0), (0, nc - 1), (ns - 1, nc - 1), (7, 2)):
        c, v, ev = o.hill_climb(rows, *start)
        assert c == c_ex and v == o_ex
        d = abs(start[0] - s_pk) + abs(start[1] - p_pk)  # moves on an L1-unimodal landscape
        assert 1 + 2 * (d + 1) <= ev <= 1 + 4 * (d + 1)
    c, v, ev = o.hill_climb(rows, s_pk, p_pk)
    assert c == c_ex and ev == 5  # itself + 4 neighbours, no move


def test_all_infeasible_and_infeasible_start_fallback():
    pb = make_problem("b200", "c10", coef_seed=7, alpha=10.0)
    o = Oracle(pb)
    F, _ = make_features(4, seed=7)
    c, v, ev = o.hill_climb([F[0], F[1]], 0, 0)
    assert c == -1 and v == -math.inf and ev >= pb.n_states * pb.n_caps
    # feasible only in the last state: a start far away in an all-infeasible plateau falls back
    pb2 = make_problem("b200", "c10", coef_seed=8, alpha=0.5, objective=1)
    ns, nc = pb2.n_states, pb2.n_caps
    ss = np.arange(ns * 2, dtype=np.int32).reshape(ns, 2)
    C = np.zeros((nc, ns * 2, 6), dtype=np.float32)
    for p in range(nc):
        C[p, ss[ns - 1], 5] = 0.95 - 0.01 * abs(p - 2)
    pb2.state_slice, pb2.slices = ss, [(0, 0)] * (ns * 2)
    pb2.coef_c, pb2.coef_d = C, np.zeros((nc, ns * 2, 3), dtype=np.float32)
    o2 = Oracle(pb2)
    c, v, ev = o2.hill_climb([F[0], F[1]], 0, 0)
    # the first start whose climb ends feasible is (ns-2, 0): it steps into the last
    # state and climbs along the caps to the peak
    assert c == (ns - 1) * nc + 2 and abs(v - 1.9) < 1e-6


def test_hill_range_matches_per_set():
    pb = make_problem("b200", "c21", coef_seed=9, alpha=0.4)
    F, _ = make_features(12, seed=9)
    o = Oracle(pb)
    cfg, obj, ev = o.hill_range(F, 0, pb.n_caps - 1)
    from oracle import unrank
    for sid in range(len(cfg)):
        rows = [F[p] for p in unrank(12, 2, sid)]
        c, v, e = o.hill_climb(rows, 0, pb.n_caps - 1)
        assert (c, e) == (cfg[sid], ev[sid]) and (v == obj[sid] or (c < 0 and obj[sid] == -math.inf))

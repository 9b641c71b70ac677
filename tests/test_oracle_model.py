"""Pins of the oracle's basis functions, model, metrics and per-set search.

Each test fixes the oracle against something other than itself: values the
paper / SPEC print, a hand derivation with exact dyadic arithmetic
(tests/golden/hand_pair_example.json), closed forms and invariants.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle import Oracle
from synth import Problem, make_problem, make_features


def _problem_from_json(p, objective, alpha):
    return Problem(name="hand", n_slots=p["n_slots"], gpcs_total=p["gpcs_total"],
                   state_gpcs=np.array(p["state_gpcs"], dtype=np.int32),
                   state_mem=np.array(p["state_mem"], dtype=np.int32),
                   state_slice=np.array(p["state_slice"], dtype=np.int32),
                   slices=[(0, 0)] * len(p["coef_c"][0]),
                   caps_w=np.array(p["caps_w"], dtype=np.float32),
                   coef_c=np.array(p["coef_c"], dtype=np.float32),
                   coef_d=np.array(p["coef_d"], dtype=np.float32),
                   objective=objective, alpha=alpha)


# ---- basis (Table `functions`) --------------------------------

def test_basis_spec_examples(golden):
    g = golden("spec_basis_examples.json")
    for ex in g["h_examples"]:
        assert np.allclose(oracle.basis_h(ex["f"]), ex["h"], rtol=0, atol=1e-12), ex["cite"]
    for ex in g["j_examples"]:
        f = [50, 0, ex["f3"], ex["f4"], 0, 0, 0, 0]
        assert np.allclose(oracle.basis_j(f), ex["j"], rtol=0, atol=1e-12), ex["cite"]


def test_basis_hand_example(golden):
    g = golden("hand_pair_example.json")
    for name in ("A", "B"):
        f = g["features"][name]
        assert list(oracle.basis_h(f)) == g["basis_by_hand"]["H_" + name]
        assert list(oracle.basis_j(f)) == g["basis_by_hand"]["J_" + name]


def test_basis_identity_h1_plus_h2():
    """h1 + h2 = f1/100 for every valid profile (Table `functions` algebra)."""
    F, _ = make_features(300, seed=7)
    for f in F:
        h = oracle.basis_h(f)
        assert abs(h[0] + h[1] - float(f[0]) / 100.0) < 1e-15
        assert h[5] == 1.0 and oracle.basis_j(f)[2] == 1.0


def test_degenerate_and_range_validation(golden):
    g = golden("spec_basis_examples.json")
    bad = np.array([g["degenerate"][0]["f"]], dtype=np.float32)
    assert Oracle.validate_features(bad)[0] == oracle.E_DEGENERATE_PROFILE
    ok = np.array([[80, 40, 30, 60, 50, 10, 0, 0]], dtype=np.float32)
    assert Oracle.validate_features(ok)[0] == oracle.OK
    for k, v in [(0, 101.0), (3, -1.0), (4, float("nan")), (2, float("inf"))]:
        b = ok.copy()
        b[0, k] = v
        assert Oracle.validate_features(b)[0] == oracle.E_RANGE
    b = ok.copy()
    b[0, 5:8] = [50, 40, 20]  # F6+F7+F8 = 110 > 100
    assert Oracle.validate_features(b)[0] == oracle.E_RANGE
    b = ok.copy()
    b[0, 0] = 0.01  # F1 <= 0.01 is degenerate (boundary inclusive)
    assert Oracle.validate_features(b)[0] == oracle.E_DEGENERATE_PROFILE
    b[0, 0] = np.nextafter(np.float32(0.01), np.float32(1))
    assert Oracle.validate_features(b)[0] == oracle.OK
    # first bad job wins; jobs index rows
    two = np.vstack([ok, bad])
    assert Oracle.validate_features(two, np.array([0, 1, 0], dtype=np.int32))[0] == oracle.E_DEGENERATE_PROFILE
    assert Oracle.validate_features(two, np.array([0, 2], dtype=np.int32))[0] == oracle.E_ARG


# ---- model -----------------------------------------------

def _tiny(n_slots=1, c=(0, 0, 0, 0, 0, 0.8), d=(0, 0, 0), objective=2, alpha=0.0):
    st = np.ones((1, n_slots), dtype=np.int32)
    st[0, 0] = 8 - (n_slots - 1)
    return Problem(name="t", n_slots=n_slots, gpcs_total=8, state_gpcs=st, state_mem=np.zeros(1, np.int32),
                   state_slice=np.zeros((1, n_slots), np.int32), slices=[(8, 0)],
                   caps_w=np.array([100.0], np.float32), coef_c=np.array([[c]], np.float32),
                   coef_d=np.array([[d]], np.float32), objective=objective, alpha=alpha)


def test_constant_only_model(golden):
    g = golden("spec_model_metric_examples.json")["constant_only"]
    o = Oracle(_tiny(c=g["c"]))
    F, _ = make_features(20, seed=3)
    for f in F:
        assert o.rperf([f], 0, 0, 0) == pytest.approx(g["rperf"], abs=1e-7)  # 0.8f


def test_hand_dot_product(golden):
    """c.H = 0.7 and partner term -0.15 give 0.55 (the interference term is added)."""
    g = golden("spec_model_metric_examples.json")["hand_dot"]
    # H of f=(80,40,30,60,50,10,0,0) is (0.7,0.1,0.5,0.6,0.5,1): c = e1 gives c.H = 0.7.
    # J of the partner (f3=30, f4=60) is (0.3,0.6,1): d = (-0.5, 0, 0) gives -0.15.
    o = Oracle(_tiny(n_slots=2, c=(1, 0, 0, 0, 0, 0), d=(-0.5, 0, 0)))
    f = np.array([80, 40, 30, 60, 50, 10, 0, 0], np.float32)
    assert o.rperf([f, f], 0, 0, 0) == pytest.approx(g["rperf"], abs=1e-7)


def test_solo_ignores_d():
    """P:L468 / SPEC.md L263: with no partners the interference term vanishes."""
    F, _ = make_features(10, seed=4)
    a = Oracle(_tiny(c=(0.3, -0.2, 0.01, 0.1, -0.4, 0.9), d=(0, 0, 0)))
    b = Oracle(_tiny(c=(0.3, -0.2, 0.01, 0.1, -0.4, 0.9), d=(5, -7, 11)))
    for f in F:
        assert a.rperf([f], 0, 0, 0) == b.rperf([f], 0, 0, 0)


def test_normalisation_baseline_is_exactly_one():
    """RPerf is normalised to the exclusive, unpartitioned, uncapped run.
    The baseline row (G_full, P_max) is C = e6, D = 0 (R11) -> RPerf == 1.0 exactly."""
    pb = make_problem("solo", "c10", coef_seed=11)
    o = Oracle(pb)
    F, _ = make_features(200, seed=12)
    top = pb.n_caps - 1
    for f in F:
        assert o.rperf([f], 0, 0, top) == 1.0
    # and through the search: the full-chip solo job at P_max has obj 1/P_max
    cfgs, objs = o.score_range(F)
    obj_all, _, thr, _, _ = o.eval_set([F[0]])
    assert thr[top] == 1.0


def test_metrics_examples(golden):
    """Throughput = sum, Fairness = min via a model whose RPerf equals the constant."""
    g = golden("spec_model_metric_examples.json")
    for ex in g["throughput"] + g["fairness"]:
        r = ex["rperfs"]
        pb = Problem(name="m", n_slots=2, gpcs_total=8, state_gpcs=np.array([[4, 4]], np.int32),
                     state_mem=np.zeros(1, np.int32), state_slice=np.array([[0, 1]], np.int32),
                     slices=[(4, 0), (4, 0)], caps_w=np.array([1.0], np.float32),
                     coef_c=np.array([[[0, 0, 0, 0, 0, r[0]], [0, 0, 0, 0, 0, r[1]]]], np.float32),
                     coef_d=np.zeros((1, 2, 3), np.float32), objective=1, alpha=0.0)
        F, _ = make_features(2, seed=1)
        obj, fair, thr, feas, rp = Oracle(pb).eval_set([F[0], F[1]])
        want_thr = float(np.float32(r[0])) + float(np.float32(r[1]))
        want_fair = min(float(np.float32(r[0])), float(np.float32(r[1])))
        assert thr[0] == pytest.approx(want_thr, abs=1e-12)
        assert fair[0] == pytest.approx(want_fair, abs=1e-12)
        key = "throughput" if ex in g["throughput"] else "fairness"
        got = thr[0] if key == "throughput" else fair[0]
        assert got == pytest.approx(ex["value"], abs=1e-7), ex["cite"]


# ---- the hand-derived pair (exact dyadic arithmetic) -----------------------

@pytest.mark.parametrize("case", range(5))
def test_hand_pair_choices(golden, case):
    g = golden("hand_pair_example.json")
    ch = g["choices_by_hand"][case]
    pb = _problem_from_json(g["problem"], ch["objective"], ch["alpha"])
    o = Oracle(pb)
    A = np.array(g["features"]["A"], np.float32)
    B = np.array(g["features"]["B"], np.float32)
    obj, fair, thr, feas, rp = o.eval_set([A, B])
    for row in g["per_config_by_hand"]:
        c = row["cfg"]
        assert list(rp[c]) == row["rperf"]          # exact: every value is dyadic
        assert thr[c] == row["throughput"] and fair[c] == row["fairness"]
    cfg, ob = o.best_config([A, B])
    assert cfg == ch["cfg"], ch["why"]
    if ch["obj"] is None:
        assert ob == -math.inf
    else:
        assert ob == pytest.approx(ch["obj"], rel=1e-15)


def test_hand_pair_mirror(golden):
    """Swapping the queue order swaps the slots."""
    g = golden("hand_pair_example.json")
    pb = _problem_from_json(g["problem"], 2, 0.0)
    A = np.array(g["features"]["A"], np.float32)
    B = np.array(g["features"]["B"], np.float32)
    _, _, _, _, rp_ab = Oracle(pb).eval_set([A, B])
    _, _, _, _, rp_ba = Oracle(pb).eval_set([B, A])
    want = {0: [0.375, 0.5], 1: [0.375, 0.75], 2: [0.75, 0.25], 3: [0.5625, 0.625]}
    for c, r in want.items():
        assert list(rp_ba[c]) == r
    # state s of [B,A] is state 1-s of [A,B] with slots reversed
    for s in range(2):
        for p in range(2):
            assert list(rp_ba[s * 2 + p]) == list(rp_ab[(1 - s) * 2 + p][::-1])


# ---- search-space and argmax semantics ----------------------------------

def test_paper_search_space(golden):
    g = golden("paper_search_space.json")
    pb = make_problem("a100_paper", "a100_paper", coef_seed=1)
    assert list(pb.caps_w) == g["caps_w"]
    assert pb.n_states == 4 and pb.gpcs_total == g["usable_gpcs"]
    for (a, b, m), gp, mem in zip(g["states"], pb.state_gpcs, pb.state_mem):
        assert (a, b) == tuple(gp) and mem == (0 if m == "shared" else 1)
    assert pb.n_configs == g["n_candidates_problem2"]
    o = Oracle(pb)
    F, _ = make_features(2, seed=5, classes=("TI", "MI"))
    assert len(o.eval_set([F[0], F[1]])[0]) == 24
    p1 = make_problem("a100_paper", "a100_230", coef_seed=1, objective=1)
    assert Oracle(p1).n_configs == g["n_candidates_problem1"]


def test_alpha_extremes():
    """alpha = 0 is vacuous for positive RPerf; alpha = 10 is infeasible (L349)."""
    pb = make_problem("b200", "c10", coef_seed=9, alpha=0.0)
    F, _ = make_features(12, seed=9)
    o = Oracle(pb)
    for a, b in [(0, 1), (3, 7), (10, 11)]:
        obj, fair, thr, feas, rp = o.eval_set([F[a], F[b]])
        assert np.array_equal(feas, (rp > 0).all(axis=1))
    pb.alpha = 10.0
    o = Oracle(pb)
    st, sid, cfg, ob = o.best_set(F)
    assert st == oracle.INFEASIBLE and sid == -1 and cfg == -1


def test_dominance_picks_dominating_state():
    """A state whose coefficients dominate every other state wins.
    Full (state, slot) keying (reading R1) so the boost touches one state only."""
    pb = make_problem("b200", "c10", coef_seed=21, alpha=0.2)
    full = pb.state_slice.reshape(-1)
    pb.coef_c = pb.coef_c[:, full].copy()
    pb.coef_d = pb.coef_d[:, full].copy()
    pb.state_slice = np.arange(2 * pb.n_states, dtype=np.int32).reshape(pb.n_states, 2)
    pb.slices = [pb.slices[i] for i in full]
    F, _ = make_features(6, seed=21)
    for win in (0, 9, 13):
        C = pb.coef_c.copy()
        C[:, 2 * win:2 * win + 2, 5] += 5.0
        q = make_problem("b200", "c10", coef_seed=21, alpha=0.2)
        q.coef_c, q.coef_d, q.state_slice, q.slices = C, pb.coef_d, pb.state_slice, pb.slices
        cfg, _ = Oracle(q).best_config([F[0], F[1]])
        assert cfg // q.n_caps == win


def test_rescaling_and_problem1_equals_problem2_on_one_cap():
    """argmax is invariant under positive rescaling; Problem 1 at P equals
    Problem 2 restricted to {P}."""
    F, _ = make_features(10, seed=31)
    base = make_problem("b200", "c1_900", coef_seed=31, objective=1, alpha=0.2)
    p2 = make_problem("b200", "c1_900", coef_seed=31, objective=2, alpha=0.2)
    scaled = make_problem("b200", "c1_900", coef_seed=31, objective=1, alpha=0.4)
    scaled.coef_c = base.coef_c * 2  # exact power-of-two scaling
    scaled.coef_d = base.coef_d * 2
    for a, b in itertools.combinations(range(10), 2):
        c1, o1 = Oracle(base).best_config([F[a], F[b]])
        c2, o2 = Oracle(p2).best_config([F[a], F[b]])
        c3, o3 = Oracle(scaled).best_config([F[a], F[b]])
        assert c1 == c2 == c3
        if c1 >= 0:
            assert o2 == pytest.approx(o1 / 900.0, rel=1e-15) and o3 == 2 * o1


def test_duplicate_jobs_tie_to_lowest_config():
    """A job paired with its own copy makes mirrored states (g,8-g)/(8-g,g) exact ties;
    the canonical rule keeps the lower config id."""
    pb = make_problem("b200", "c10", coef_seed=41, alpha=0.2)
    o = Oracle(pb)
    F, _ = make_features(30, seed=41)
    n_mirror_wins = 0
    for f in F:
        obj, fair, thr, feas, rp = o.eval_set([f, f])
        cfg, best = o.best_config([f, f])
        assert cfg >= 0
        s, p = divmod(cfg, pb.n_caps)
        g0, g1 = pb.state_gpcs[s]
        mirror = [t for t in range(pb.n_states) if tuple(pb.state_gpcs[t]) == (g1, g0)
                  and pb.state_mem[t] == pb.state_mem[s]][0]
        mc = mirror * pb.n_caps + p
        assert obj[mc] == obj[cfg]            # exact tie
        assert cfg <= mc                      # lowest config id wins
        n_mirror_wins += mc != cfg
    assert n_mirror_wins > 0


def test_problem_validation_codes():
    pb = make_problem("b200", "c10", coef_seed=1)
    assert Oracle(pb).validate()[0] == oracle.OK
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.state_gpcs = bad.state_gpcs.copy()
    bad.state_gpcs[3, 0] += 1                  # split sums to 9, not 8
    assert Oracle(bad).validate()[0] == oracle.E_INVALID_ALLOCATION
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.state_gpcs = np.array([[8, 0]] + [[4, 4]] * 13, np.int32)  # a slot with 0 GPCs
    assert Oracle(bad).validate()[0] == oracle.E_INVALID_ALLOCATION
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.state_slice = bad.state_slice.copy()
    bad.state_slice[0, 1] = 99
    assert Oracle(bad).validate()[0] == oracle.E_UNKNOWN_KEY
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.caps_w = bad.caps_w[::-1].copy()
    assert Oracle(bad).validate()[0] == oracle.E_INVALID_ALLOCATION
    bad = make_problem("b200", "c10", coef_seed=1, alpha=-0.1)
    assert Oracle(bad).validate()[0] == oracle.E_ARG
    bad = make_problem("b200", "c10", coef_seed=1, objective=3)
    assert Oracle(bad).validate()[0] == oracle.E_ARG
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.state_mem = bad.state_mem.copy()
    bad.state_mem[2] = 2
    assert Oracle(bad).validate()[0] == oracle.E_INVALID_ALLOCATION


# ---- the hand-derived triple (exact dyadic arithmetic; n_slots = 3) --------
# Pins orc_rperf for three applications: slot i sums the J of BOTH partners
# under the D of its OWN slice (reading R14).

def test_hand_triple_basis(golden):
    g = golden("hand_triple_example.json")
    for name in ("A", "B", "C"):
        f = g["features"][name]
        assert list(oracle.basis_h(f)) == g["basis_by_hand"]["H_" + name]
        assert list(oracle.basis_j(f)) == g["basis_by_hand"]["J_" + name]


@pytest.mark.parametrize("case", range(5))
def test_hand_triple_choices(golden, case):
    g = golden("hand_triple_example.json")
    ch = g["choices_by_hand"][case]
    pb = _problem_from_json(g["problem"], ch["objective"], ch["alpha"])
    assert Oracle(pb).validate()[0] == oracle.OK
    o = Oracle(pb)
    rows = [np.array(g["features"][k], np.float32) for k in g["queue"]]
    obj, fair, thr, feas, rp = o.eval_set(rows)
    for row in g["per_config_by_hand"]:
        c = row["cfg"]
        assert list(rp[c]) == row["rperf"], c      # exact: every value is dyadic
        assert thr[c] == row["throughput"] and fair[c] == row["fairness"]
    for s in range(3):  # one scalar RPerf entry point agrees with the set evaluation
        for p in range(2):
            for i in range(3):
                assert o.rperf(rows, i, s, p) == rp[s * 2 + p][i]
    cfg, ob = o.best_config(rows)
    assert cfg == ch["cfg"], ch["why"]
    if ch["obj"] is None:
        assert ob == -math.inf
    else:
        assert ob == pytest.approx(ch["obj"], rel=1e-15)


def test_hand_triple_queue_order(golden):
    """Queue [C, A, B] puts C in slot 0 (slot i <- i-th smallest queue position, reading R15):
    state 0 then gives C slice 0, A slice 1, B slice 2; by hand from the golden's terms:
    C: .5 + D0.J_A + D0.J_B = .5 - .0625 - .1875 = .25; A: .625 + D1.J_C + D1.J_B =
    .625 - .1875 - .0625 = .375; B: .375 + D2.J_C + D2.J_A = .375 - .21875 - .15625 = 0."""
    g = golden("hand_triple_example.json")
    pb = _problem_from_json(g["problem"], 2, 0.0)
    rows = [np.array(g["features"][k], np.float32) for k in ("C", "A", "B")]
    _, _, _, _, rp = Oracle(pb).eval_set(rows)
    assert list(rp[0]) == [0.25, 0.375, 0.0]


def test_fp32_tensor_sum_reading():
    """Reading R24: F6+F7+F8 <= 100 is decided on the FP32 sum (F6+F7)+F8 --
    the precision of the FP32 inputs and of the CUDA path's decision (a status is an
    integer decided by floating point: both sides decide it in the same precision).
    These three FP32 values sum to exactly 100.0 in FP32 but to 100.0000038 in FP64:
    valid under the reading."""
    f6, f7, f8 = np.float32(33.33333206176758), np.float32(33.33333206176758), np.float32(33.33333969116211)
    assert np.float32(np.float32(f6 + f7) + f8) == np.float32(100.0)
    assert float(f6) + float(f7) + float(f8) > 100.0
    row = np.array([[90, 40, 30, 60, 50, f6, f7, f8]], np.float32)
    assert Oracle.validate_features(row)[0] == oracle.OK
    row[0, 7] = np.nextafter(f8, np.float32(200))
    assert Oracle.validate_features(row)[0] == oracle.E_RANGE

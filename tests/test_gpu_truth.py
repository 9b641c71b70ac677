"""GPU worst / proposal / best (cosched_evaluate_truth, NEXT #3) vs the FP64 oracle
(oracle/evaluate.py) on seeded queues.

Bar: per-set ground-truth values within 1e-5 relative (FP32 simulator vs FP64);
best / worst are values, so argmax ties do not matter; a fairness decision may
differ only within 1e-5 of alpha; summary counts equal up to those near-threshold
sets, geometric means within 1e-5 relative.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import evaluate as ev  # noqa: E402
from synth import bench_config, make_features, make_problem  # noqa: E402
from synth.ground_truth import A100, B200  # noqa: E402

TOL = 1e-5


@pytest.fixture(scope="module")
def cs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03838_b200 as cs
    return cs


def _close(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    return both_inf | (np.abs(a - b) <= TOL * np.abs(b) + 1e-12)


def _fairness_margin(pb, F, model, sid, n):
    """min over configs of |truth Fairness - alpha| for set sid (FP64, oracle/evaluate.py's truth)."""
    from oracle import unrank
    from synth.ground_truth import true_rperf
    rows = [F[p:p + 1] for p in unrank(n, pb.n_slots, sid)]
    alpha = float(np.float32(pb.alpha))
    m = math.inf
    for st in range(pb.n_states):
        gp = tuple(int(g) for g in pb.state_gpcs[st])
        for p in range(pb.n_caps):
            r = true_rperf(model, rows, gp, int(pb.state_mem[st]), float(pb.caps_w[p]))
            m = min(m, abs(float(np.min(r)) - alpha))
    return m


def _run(cs, pb, F, model, mode=0):
    s = cs.Scheduler(pb)
    if mode:
        s.set_search(1, 0, 0)
    Fd = torch.from_numpy(F).cuda()
    obj, cfg = s.score_all(Fd)
    (po, pf, best, worst), sm = s.evaluate_truth(Fd, model)
    torch.cuda.synchronize()
    return cfg.cpu().numpy(), [t.cpu().numpy() for t in (po, pf, best, worst)], sm


@pytest.mark.parametrize("table,caps,n,model", [("b200", "c10", 150, B200), ("b200_3way", "c10", 30, B200),
                                                ("a100_paper", "a100_paper", 60, A100)])
def test_parity(cs, table, caps, n, model):
    pb = make_problem(table, caps, coef_seed=101, alpha=0.2)
    F, _ = make_features(n, seed=102)
    cfg, (po, pf, best, worst), sm = _run(cs, pb, F, model)
    opo, opf, obest, oworst = ev.worst_prop_best(pb, F, cfg, model)
    alpha = float(np.float32(pb.alpha))
    near = np.abs(np.where(np.isfinite(opf), opf, 0) - alpha) <= TOL  # fairness decisions may flip here
    assert np.all(_close(po, opo)) and np.all(_close(pf, opf))
    # best / worst can differ only on sets whose truth has a config with Fairness
    # within TOL of alpha (FP32 vs FP64 may decide that config's feasibility
    # differently): every mismatching set is checked for exactly that
    ok = _close(best, obest) & _close(worst, oworst)
    assert ok.mean() > 0.999, ok.mean()
    for sid in np.nonzero(~ok)[0]:
        assert _fairness_margin(pb, F, model, int(sid), n) <= TOL, sid
    osm = ev.summary(pb, cfg, opo, opf, obest, oworst)
    assert abs(sm["n_compared"] - osm["n_compared"]) <= int((~ok).sum())
    assert abs(sm["n_violations"] - osm["n_violations"]) <= int(near.sum())
    assert abs(sm["geomean_prop_over_best"] - osm["geomean_prop_over_best"]) <= 1e-4
    assert abs(sm["geomean_worst_over_best"] - osm["geomean_worst_over_best"]) <= 1e-4
    assert sm["geomean_worst_over_best"] <= sm["geomean_prop_over_best"] <= 1.0 + 1e-6


def test_calibrated_pipeline_at_c3_scale(cs):
    """The paper's workflow end to end on the GPU: calibrate C, D on the synthetic GPU
    (cosched_fit), search a 1,000-job queue exhaustively and by hill climbing, evaluate both
    against the ground truth. The calibrated proposals land near the truth optimum
    (geomean proposal/best well above worst/best), the evaluation follows the active search
    mode, and sampled per-set values match the ground truth."""
    from oracle import unrank
    from synth.ground_truth import make_training_set, true_rperf
    pb = make_problem("b200", "c10", coef_seed=104, alpha=0.2)
    Ft, _ = make_features(1000, seed=105)
    ts = make_training_set(Ft, pb, n_corun=100000, seed=106, noise=0.0)
    d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()
    r = cs.fit(d(Ft, np.float32), pb.n_slices, pb.n_caps, d(ts.solo_app, np.int32), d(ts.solo_key, np.int32),
               d(ts.solo_rperf, np.float32), d(ts.co_app, np.int32), d(ts.co_partners, np.int32),
               d(ts.co_key, np.int32), d(ts.co_rperf, np.float32)).cpu()
    pb.coef_c = r.coef_c.astype(np.float32)
    pb.coef_d = r.coef_d.astype(np.float32)
    F, _ = make_features(1000, seed=107)
    cfg_e, (po_e, *_), sm_e = _run(cs, pb, F, B200, mode=0)
    cfg_h, (po_h, *_), sm_h = _run(cs, pb, F, B200, mode=1)
    assert sm_e["n_compared"] > 0.5 * len(cfg_e)
    assert sm_e["geomean_prop_over_best"] > 0.8
    assert sm_e["geomean_prop_over_best"] > sm_e["geomean_worst_over_best"] + 0.2
    assert abs(sm_h["geomean_prop_over_best"] - sm_e["geomean_prop_over_best"]) < 0.1
    for cfg, po in ((cfg_e, po_e), (cfg_h, po_h)):
        for sid in np.arange(0, len(cfg), 9973)[:30]:
            c = int(cfg[sid])
            if c < 0:
                continue
            s, p = divmod(c, pb.n_caps)
            rows = [F[q][None] for q in unrank(F.shape[0], 2, int(sid))]
            rt = true_rperf(B200, rows, tuple(pb.state_gpcs[s]), int(pb.state_mem[s]), float(pb.caps_w[p]))[:, 0]
            assert abs(po[sid] - rt.sum() / float(pb.caps_w[p])) <= TOL * abs(po[sid])


def test_errors(cs):
    pb = make_problem("b200", "c10", coef_seed=103)
    F, _ = make_features(20, seed=103)
    s = cs.Scheduler(pb)
    Fd = torch.from_numpy(F).cuda()
    with pytest.raises(cs.CoschedError):  # before score_all
        s.evaluate_truth(Fd, B200)
    s.score_all(Fd)

    class Bad:
        g_full, n_modules, modules, w_base, w_gpc, kappa, f_min, p_max = 4, 8, {}, 200.0, 110.0, 0.6, 0.1, 1000.0
    with pytest.raises(cs.CoschedError):  # a state gives 7 GPCs > g_full = 4
        s.evaluate_truth(Fd, Bad)

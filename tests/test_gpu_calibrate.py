"""GPU calibration (cosched_fit through the C-ABI) vs the FP64 least-squares oracle
(oracle/calibrate.py) on seeded synthetic training sets.

Bar: per-key statuses and sample counts bit-exact; coefficients within 1e-6
relative (+1e-9 absolute) of the oracle -- normal equations (GPU) and SVD
least squares (oracle) differ by O(cond(X)^2 * 2^-52), far below that for
the conditioning of these designs; exact recovery of known coefficients
within 1e-6 relative (SPEC acceptance 1).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import calibrate as cal  # noqa: E402
from synth import make_features, make_problem  # noqa: E402
from synth.generator import SplitMix64  # noqa: E402
from synth.ground_truth import make_training_set  # noqa: E402


@pytest.fixture(scope="module")
def cs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03838_b200 as cs
    return cs


def _gpu_fit(cs, F, ts, n_slices, n_caps):
    d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()
    co = len(ts.co_app) > 0
    r = cs.fit(d(F, np.float32), n_slices, n_caps, d(ts.solo_app, np.int32), d(ts.solo_key, np.int32),
               d(ts.solo_rperf, np.float32),
               d(ts.co_app, np.int32) if co else None, d(ts.co_partners, np.int32) if co else None,
               d(ts.co_key, np.int32) if co else None, d(ts.co_rperf, np.float32) if co else None)
    torch.cuda.synchronize()
    return r.cpu()


def _compare(g, o, n_keys):
    C, D, cst, dst, ccnt, dcnt, crms, drms = o
    assert np.array_equal(g.status[:, 0], cst), (g.status[:, 0], cst)
    assert np.array_equal(g.status[:, 1], dst), (g.status[:, 1], dst)
    assert np.array_equal(g.count[:, 0], ccnt) and np.array_equal(g.count[:, 1], dcnt)
    gc = g.coef_c.reshape(n_keys, 6)
    gd = g.coef_d.reshape(n_keys, 3)
    ok_c = cst == cal.FIT_OK
    ok_d = dst == cal.FIT_OK
    assert np.allclose(gc[ok_c], C[ok_c], rtol=1e-6, atol=1e-9), np.abs(gc[ok_c] - C[ok_c]).max()
    assert np.allclose(gd[ok_d], D[ok_d], rtol=1e-6, atol=1e-9), np.abs(gd[ok_d] - D[ok_d]).max()
    assert np.all(gc[~ok_c] == 0) and np.all(gd[~ok_d] == 0)
    assert np.allclose(g.rms[ok_c, 0], crms[ok_c], rtol=1e-5, atol=1e-12)
    assert np.allclose(g.rms[ok_d, 1], drms[ok_d], rtol=1e-5, atol=1e-12)


def test_exact_recovery(cs):
    """Noiseless targets from known C*, D* (computed with the oracle's basis): the GPU fit
    recovers them within 1e-6 relative and matches the oracle fit."""
    from synth.ground_truth import TrainingSet
    F, _ = make_features(80, seed=21)
    H, J = cal.basis_rows(F)
    n_slices, n_caps = 3, 2
    nk = n_slices * n_caps
    Cs = -1 + 2 * SplitMix64(22).uniform(nk * 6).reshape(nk, 6)
    Ds = -0.5 * SplitMix64(23).uniform(nk * 3).reshape(nk, 3)
    app = np.tile(np.arange(80), nk).astype(np.int32)
    key = np.repeat(np.arange(nk), 80).astype(np.int32)
    y = np.einsum("ij,ij->i", H[app], Cs[key])
    rng = SplitMix64(24)
    m = 3000
    a = (rng.uniform(m) * 80).astype(np.int64)
    b = (a + 1 + (rng.uniform(m) * 79).astype(np.int64)) % 80
    k = (rng.uniform(m) * nk).astype(np.int64)
    yc = np.einsum("ij,ij->i", H[a], Cs[k]) + np.einsum("ij,ij->i", J[b], Ds[k])
    ts = TrainingSet(n_slices, n_caps, 2, app, key, y.astype(np.float32), a.astype(np.int32),
                     b[:, None].astype(np.int32), k.astype(np.int32), yc.astype(np.float32))
    g = _gpu_fit(cs, F, ts, n_slices, n_caps)
    # float32 targets: recovery to the rounding of y (2^-24 relative), i.e. ~1e-6 on the coefficients
    assert (g.status == 0).all()
    assert np.max(np.abs(g.coef_c.reshape(nk, 6) - Cs)) < 1e-5
    assert np.max(np.abs(g.coef_d.reshape(nk, 3) - Ds)) < 1e-5
    _compare(g, cal.fit(F, ts, nk), nk)


@pytest.mark.parametrize("table,caps,n,nco,noise", [("b200", "c10", 200, 20000, 0.01),
                                                     ("b200", "c21", 500, 50000, 0.0),
                                                     ("b200_3way", "c10", 150, 20000, 0.01),
                                                     ("a100_paper", "a100_paper", 60, 3000, 0.01)])
def test_parity_on_synthetic_gpu(cs, table, caps, n, nco, noise):
    pb = make_problem(table, caps, coef_seed=31)
    F, _ = make_features(n, seed=32)
    ts = make_training_set(F, pb, n_corun=nco, seed=33, noise=noise)
    nk = pb.n_slices * pb.n_caps
    g = _gpu_fit(cs, F, ts, pb.n_slices, pb.n_caps)
    _compare(g, cal.fit(F, ts, nk), nk)


def test_statuses_insufficient_rank_missing(cs):
    """Keys with too few samples, a rank-deficient partner design and co-runs on a key without
    C get the oracle's statuses; keys without samples report NO_SAMPLES."""
    from synth.ground_truth import TrainingSet
    F, _ = make_features(40, seed=41)
    # key 0: 30 solo samples (fits); key 1: 5 solo samples (insufficient); key 2: none;
    # co-runs: key 0 with identical partners (rank 1), key 1 (missing C)
    app = np.concatenate([np.arange(30), np.arange(5)]).astype(np.int32)
    key = np.concatenate([np.zeros(30), np.ones(5)]).astype(np.int32)
    y = (0.5 + 0.01 * np.arange(35)).astype(np.float32)
    ca = np.arange(20).astype(np.int32)
    cp = np.full((20, 1), 7, dtype=np.int32)
    ck = np.concatenate([np.zeros(10), np.ones(10)]).astype(np.int32)
    cy = np.linspace(0.3, 0.6, 20).astype(np.float32)
    ts = TrainingSet(3, 1, 2, app, key, y, ca, cp, ck, cy)
    g = _gpu_fit(cs, F, ts, 3, 1)
    o = cal.fit(F, ts, 3)
    assert list(g.status[:, 0]) == [cal.FIT_OK, cal.FIT_INSUFFICIENT, cal.FIT_NO_SAMPLES]
    assert list(g.status[:, 1]) == [cal.FIT_RANK_DEFICIENT, cal.FIT_MISSING_C, cal.FIT_NO_SAMPLES]
    _compare(g, o, 3)


def test_invalid_inputs(cs):
    from synth.ground_truth import TrainingSet
    F, _ = make_features(20, seed=51)
    app = np.arange(20, dtype=np.int32)
    good = TrainingSet(2, 1, 2, app, np.zeros(20, np.int32), np.ones(20, np.float32),
                       np.zeros(0, np.int32), np.zeros((0, 1), np.int32), np.zeros(0, np.int32),
                       np.zeros(0, np.float32))
    _gpu_fit(cs, F, good, 2, 1)
    bad_key = TrainingSet(2, 1, 2, app, np.full(20, 5, np.int32), np.ones(20, np.float32),
                          good.co_app, good.co_partners, good.co_key, good.co_rperf)
    with pytest.raises(cs.CoschedError) as e:
        _gpu_fit(cs, F, bad_key, 2, 1)
    assert e.value.status == 12
    Fd = F.copy()
    Fd[3, 0] = 0.005  # F1 <= 0.01 %
    with pytest.raises(cs.CoschedError) as e:
        _gpu_fit(cs, Fd, good, 2, 1)
    assert e.value.status == 13
    Fr = F.copy()
    Fr[4, 2] = 101.0
    with pytest.raises(cs.CoschedError) as e:
        _gpu_fit(cs, Fr, good, 2, 1)
    assert e.value.status == 14


def test_deterministic_and_order_independent(cs):
    pb = make_problem("b200", "c10", coef_seed=61)
    F, _ = make_features(150, seed=62)
    ts = make_training_set(F, pb, n_corun=20000, seed=63, noise=0.01)
    a = _gpu_fit(cs, F, ts, pb.n_slices, pb.n_caps)
    b = _gpu_fit(cs, F, ts, pb.n_slices, pb.n_caps)
    assert np.array_equal(a.coef_c, b.coef_c) and np.array_equal(a.coef_d, b.coef_d)
    perm = np.argsort(SplitMix64(64).uniform(len(ts.solo_app)))
    ts.solo_app, ts.solo_key, ts.solo_rperf = ts.solo_app[perm], ts.solo_key[perm], ts.solo_rperf[perm]
    c = _gpu_fit(cs, F, ts, pb.n_slices, pb.n_caps)
    assert np.allclose(a.coef_c, c.coef_c, rtol=1e-11, atol=1e-13)


def test_fitted_table_drives_the_search(cs):
    """Calibrate on the synthetic GPU, then search with the fitted (FP32) table: the search
    matches the oracle run with the same table (the offline -> online workflow)."""
    from oracle import Oracle
    from parity import check_sets
    pb = make_problem("b200", "c10", coef_seed=71)
    F, _ = make_features(120, seed=72)
    ts = make_training_set(F, pb, n_corun=30000, seed=73, noise=0.0)
    g = _gpu_fit(cs, F, ts, pb.n_slices, pb.n_caps)
    assert (g.status[:, 0] == 0).all() and (g.status[:, 1] != cal.FIT_RANK_DEFICIENT).all()
    pb.coef_c = g.coef_c.astype(np.float32)
    pb.coef_d = g.coef_d.astype(np.float32)
    Fq, _ = make_features(60, seed=74)
    s = cs.Scheduler(pb)
    obj, cfg = s.score_all(torch.from_numpy(Fq).cuda())
    torch.cuda.synchronize()
    obj, cfg = obj.cpu().numpy(), cfg.cpu().numpy()
    o = Oracle(pb)
    cfg_o, obj_o = o.score_range(Fq)
    mism = np.nonzero(cfg != cfg_o)[0]
    _, fails = check_sets(o, Fq, None, mism, cfg[mism], obj[mism], 60, 2)
    assert not fails, fails[:3]
    assert (cfg >= 0).mean() > 0.3

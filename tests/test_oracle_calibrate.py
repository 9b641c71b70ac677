"""Pins of the calibration oracle (oracle/calibrate.py) against what the paper and
the mathematics fix (SPEC.md fit_solo / fit_interference examples and
invariants; acceptance criteria 1-2). CPU only."""
import numpy as np
import pytest

from oracle import calibrate as cal
from synth import make_features, make_problem
from synth.generator import SplitMix64
from synth.ground_truth import A100, B200, make_training_set, true_rperf


def _rand(seed, shape, lo=-1.0, hi=1.0):
    return lo + (hi - lo) * SplitMix64(seed).uniform(int(np.prod(shape))).reshape(shape)


def _queue(n, seed, mix="paper"):
    F, _ = make_features(n, seed=seed, mix=mix)
    return F


def test_exact_recovery_solo_and_corun():
    """Noiseless data from known C*, D* is refit within 1e-6 relative, RMS < 1e-9
    (SPEC acceptance 1; one least-squares fit per (S, P))."""
    F = _queue(60, 1)
    H, J = cal.basis_rows(F)
    n_keys = 4
    Cs = _rand(11, (n_keys, 6))
    Ds = _rand(12, (n_keys, 3), -0.5, 0.0)
    rng = SplitMix64(13)
    # solo: every app on every key
    app = np.tile(np.arange(60), n_keys).astype(np.int32)
    key = np.repeat(np.arange(n_keys), 60).astype(np.int32)
    y = np.einsum("ij,ij->i", H[app], Cs[key])
    C, st, cnt, rms = cal.fit_solo(H, app, key, y, n_keys)
    assert (st == cal.FIT_OK).all() and (cnt == 60).all()
    assert np.max(np.abs(C - Cs) / np.maximum(np.abs(Cs), 1e-3)) < 1e-6
    assert np.nanmax(rms) < 1e-9
    # co-runs: subject + one partner, residual target
    m = 400
    a = (rng.uniform(m) * 60).astype(np.int64)
    b = (a + 1 + (rng.uniform(m) * 59).astype(np.int64)) % 60
    k = (rng.uniform(m) * n_keys).astype(np.int64)
    yc = np.einsum("ij,ij->i", H[a], Cs[k]) + np.einsum("ij,ij->i", J[b], Ds[k])
    D, dst, dcnt, drms = cal.fit_interference(H, J, a, b[:, None], k, yc, C, st, n_keys)
    assert (dst == cal.FIT_OK).all()
    assert np.max(np.abs(D - Ds) / np.maximum(np.abs(Ds), 1e-3)) < 1e-6
    assert np.nanmax(drms) < 1e-9


def test_residual_orthogonality_and_normal_equations():
    """At the fit the residual is orthogonal to every design column (SPEC acceptance 2),
    and an independent normal-equations solve gives the same coefficients."""
    pb = make_problem("b200", "c10", coef_seed=3)
    F = _queue(120, 2)
    ts = make_training_set(F, pb, n_corun=3000, seed=5, noise=0.01)
    n_keys = pb.n_slices * pb.n_caps
    H, J = cal.basis_rows(F)
    C, cs, _, _ = cal.fit_solo(H, ts.solo_app, ts.solo_key, ts.solo_rperf, n_keys)
    for k in (0, 7, n_keys - 1):
        idx = np.nonzero(ts.solo_key == k)[0]
        X, y = H[ts.solo_app[idx]], ts.solo_rperf[idx].astype(np.float64)
        res = y - X @ C[k]
        scale = np.abs(X).max() * np.abs(y).max() * len(idx)
        assert np.abs(X.T @ res).max() <= 1e-8 * scale
        ne = np.linalg.solve(X.T @ X, X.T @ y)
        assert np.allclose(ne, C[k], rtol=1e-7, atol=1e-9)


def test_insufficient_missing_and_rank_deficient():
    F = _queue(30, 3)
    H, J = cal.basis_rows(F)
    # 5 samples < 6 coefficients (SPEC fit_solo example)
    app = np.arange(5, dtype=np.int32)
    C, st, _, _ = cal.fit_solo(H, app, np.zeros(5, np.int32), np.ones(5), 2)
    assert st[0] == cal.FIT_INSUFFICIENT and st[1] == cal.FIT_NO_SAMPLES
    # all partners the same profile: the summed-J design has rank 1 (SPEC fit_interference example)
    app = np.arange(30, dtype=np.int32)
    Cf, cst, _, _ = cal.fit_solo(H, app, np.zeros(30, np.int32), np.ones(30), 1)
    assert cst[0] == cal.FIT_OK
    D, dst, _, _ = cal.fit_interference(H, J, app, np.full((30, 1), 4), np.zeros(30, np.int64), np.ones(30),
                                        Cf, cst, 1)
    assert dst[0] == cal.FIT_RANK_DEFICIENT
    # co-run samples on a key without C (SPEC MissingScalabilityCoefficients)
    D, dst, _, _ = cal.fit_interference(H, J, app, (app[:, None] + 1) % 30, np.ones(30, np.int64), np.ones(30),
                                        np.zeros((2, 6)), np.array([cal.FIT_OK, cal.FIT_NO_SAMPLES]), 2)
    assert dst[1] == cal.FIT_MISSING_C
    # a design column that is identically zero (no tensor work in the queue: H2 = 0)
    Fr = _queue(40, 4, mix="rodinia")
    Hr, _ = cal.basis_rows(Fr)
    assert np.all(Hr[:, 1] == 0)
    _, st, _, _ = cal.fit_solo(Hr, np.arange(40, dtype=np.int32), np.zeros(40, np.int32), np.ones(40), 1)
    assert st[0] == cal.FIT_RANK_DEFICIENT


def test_baseline_targets_one_give_e6():
    """Targets == 1 with the constant column fit C = e6 exactly (DESIGN reading c11)."""
    F = _queue(50, 6)
    H, _ = cal.basis_rows(F)
    C, st, _, rms = cal.fit_solo(H, np.arange(50, dtype=np.int32), np.zeros(50, np.int32), np.ones(50), 1)
    assert st[0] == cal.FIT_OK
    assert np.allclose(C[0], [0, 0, 0, 0, 0, 1], atol=1e-12) and rms[0] < 1e-12


def test_permutation_invariance_and_noise_bound():
    """Permuting samples changes no coefficient by more than 1e-12 (SPEC invariant);
    sigma = 0.01 noise on 50 profiles keeps ||c - c*||_inf < 0.02 (SPEC example)."""
    F = _queue(50, 7)
    H, _ = cal.basis_rows(F)
    cs = np.array([0.3, -0.2, 0.05, 0.1, -0.1, 0.9])
    rng = SplitMix64(8)
    u1, u2 = np.maximum(rng.uniform(50), 1e-300), rng.uniform(50)
    noise = 0.01 * np.sqrt(-2 * np.log(u1)) * np.cos(2 * np.pi * u2)
    y = H @ cs + noise
    app = np.arange(50, dtype=np.int32)
    C1, _, _, _ = cal.fit_solo(H, app, np.zeros(50, np.int32), y, 1)
    perm = (np.argsort(SplitMix64(9).uniform(50))).astype(np.int64)
    C2, _, _, _ = cal.fit_solo(H, app[perm], np.zeros(50, np.int32), y[perm], 1)
    assert np.abs(C1 - C2).max() <= 1e-12
    assert np.abs(C1[0] - cs).max() < 0.02


def test_ground_truth_phenomenology():
    """The synthetic GPU reproduces SPEC's hand-evaluated examples (acceptance 8):
    unscalable app at 1 GPC private @150 W -> 1.0; a tensor-heavy app at 7 GPCs
    loses performance from 250 W to 150 W; a streaming app prefers shared memory."""
    f = lambda *v: np.array([v], dtype=np.float32)
    assert true_rperf(A100, [f(10, 25, 5, 50, 15, 0, 0, 0)], (1,), 1, 150.0)[0, 0] == 1.0
    ti = f(100, 25, 10, 50, 100, 100, 0, 0)
    hi, lo = (true_rperf(A100, [ti], (7,), 0, P)[0, 0] for P in (250.0, 150.0))
    assert lo < hi
    mi = f(30, 90, 90, 10, 100, 0, 0, 0)
    assert true_rperf(A100, [mi], (3,), 0, 250.0)[0, 0] > true_rperf(A100, [mi], (3,), 1, 250.0)[0, 0]
    # the baseline point is exactly 1 for any app
    F = _queue(20, 10)
    assert np.all(true_rperf(B200, [F], (8,), 0, 1000.0) == 1.0)


def test_fit_on_ground_truth_predicts_within_band():
    """Fitting the paper's model to the synthetic GPU gives usable coefficients: the
    solo-run fit explains most of the variance (model error analogue, SPEC acceptance 7)."""
    pb = make_problem("b200", "c10", coef_seed=3)
    F = _queue(300, 11)
    ts = make_training_set(F, pb, n_corun=4000, seed=12, noise=0.0)
    n_keys = pb.n_slices * pb.n_caps
    C, D, cs, ds, cc, dc, cr, dr = cal.fit(F, ts, n_keys)
    assert (cs == cal.FIT_OK).all()
    assert np.nanmedian(cr) < 0.15

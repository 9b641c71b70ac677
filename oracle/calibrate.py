"""CPU oracle of the calibration step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may use it; the product path never imports it.

What it computes, in the paper's order (§5.1.3, §4.3
L464-465, L370; SPEC.md `fit_solo` / `fit_interference`):
  1. for every key (S, P) "independently and separately" (L465): the solo-run
     coefficients C[key] = argmin_c sum (rperf - c . H(F_app))^2 over the key's
     solo samples -- ordinary least squares (L370 "the well-known least square
     method");
  2. then, on co-run samples, the residual r = rperf - C[key] . H(F_subject) and
     D[key] = argmin_d sum (r - d . sum_{partners} J(F_partner))^2 (L661; the
     partner J's are summed, matching the model's sum_{j != i} D . J term, L458).
Basis H, J from the oracle's own FP64 basis (cosched_oracle.c).
Least squares by numpy.linalg.lstsq (SVD) -- a library primitive for the
step the paper names; numerical rank from the singular values with SPEC's
tolerance (rank-deficient iff s_min <= 1e-10 * s_max).

Per-key status: 0 fitted, 1 no samples, 2 fewer samples than coefficients,
3 rank deficient, 4 (D only) the key has no fitted C.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

from . import basis_h, basis_j

FIT_OK, FIT_NO_SAMPLES, FIT_INSUFFICIENT, FIT_RANK_DEFICIENT, FIT_MISSING_C = 0, 1, 2, 3, 4
RANK_TOL = 1e-10


def basis_rows(F: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """H [n][6] and J [n][3] of every row of F, FP64."""
    F = np.asarray(F, dtype=np.float32)
    H = np.stack([basis_h(f) for f in F]) if len(F) else np.zeros((0, 6))
    J = np.stack([basis_j(f) for f in F]) if len(F) else np.zeros((0, 3))
    return H, J


def _lstsq(X: np.ndarray, y: np.ndarray, min_rows: int):
    """(coef, status, rms) of one key."""
    n, k = X.shape
    if n == 0:
        return np.zeros(k), FIT_NO_SAMPLES, np.nan
    if n < min_rows:
        return np.zeros(k), FIT_INSUFFICIENT, np.nan
    s = np.linalg.svd(X, compute_uv=False)
    if s[-1] <= RANK_TOL * s[0]:
        return np.zeros(k), FIT_RANK_DEFICIENT, np.nan
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    res = y - X @ coef
    return coef, FIT_OK, float(np.sqrt(np.mean(res * res)))


def fit_solo(H: np.ndarray, app: np.ndarray, key: np.ndarray, y: np.ndarray, n_keys: int):
    """C [n_keys][6], status [n_keys], count [n_keys], rms [n_keys] (SPEC fit_solo)."""
    C = np.zeros((n_keys, 6))
    st = np.full(n_keys, FIT_NO_SAMPLES, dtype=np.int32)
    cnt = np.zeros(n_keys, dtype=np.int64)
    rms = np.full(n_keys, np.nan)
    y = np.asarray(y, dtype=np.float64)
    order = np.argsort(key, kind="stable")
    bounds = np.searchsorted(key[order], np.arange(n_keys + 1))
    for k in range(n_keys):
        idx = order[bounds[k]:bounds[k + 1]]
        cnt[k] = idx.size
        C[k], st[k], rms[k] = _lstsq(H[app[idx]], y[idx], 6)
    return C, st, cnt, rms


def fit_interference(H: np.ndarray, J: np.ndarray, app: np.ndarray, partners: np.ndarray, key: np.ndarray,
                     y: np.ndarray, C: np.ndarray, c_status: np.ndarray, n_keys: int):
    """D [n_keys][3], status, count, rms on the residuals of C (SPEC fit_interference)."""
    D = np.zeros((n_keys, 3))
    st = np.full(n_keys, FIT_NO_SAMPLES, dtype=np.int32)
    cnt = np.zeros(n_keys, dtype=np.int64)
    rms = np.full(n_keys, np.nan)
    y = np.asarray(y, dtype=np.float64)
    partners = np.asarray(partners).reshape(len(app), -1)
    order = np.argsort(key, kind="stable")
    bounds = np.searchsorted(key[order], np.arange(n_keys + 1))
    for k in range(n_keys):
        idx = order[bounds[k]:bounds[k + 1]]
        cnt[k] = idx.size
        if idx.size == 0:
            continue
        if c_status[k] != FIT_OK:
            st[k] = FIT_MISSING_C
            continue
        r = y[idx] - H[app[idx]] @ C[k]
        Z = np.zeros((idx.size, 3))
        for l in range(partners.shape[1]):
            Z += J[partners[idx, l]]
        D[k], st[k], rms[k] = _lstsq(Z, r, 3)
    return D, st, cnt, rms


def fit(F: np.ndarray, ts, n_keys: int):
    """Both stages: (C, D, c_status, d_status, c_count, d_count, c_rms, d_rms)."""
    H, J = basis_rows(F)
    C, cs, cc, cr = fit_solo(H, ts.solo_app, ts.solo_key, ts.solo_rperf, n_keys)
    D, ds, dc, dr = fit_interference(H, J, ts.co_app, ts.co_partners, ts.co_key, ts.co_rperf, C, cs, n_keys)
    return C, D, cs, ds, cc, dc, cr, dr

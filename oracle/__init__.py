"""CPU oracle for the exhaustive co-location search -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path
(paper_2405_03838_b200/) never imports it and must fail loudly without its
CUDA extension; it has no CPU fallback.

The arithmetic lives in cosched_oracle.c (plain C, FP64, single-threaded);
this module only compiles it with gcc and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cosched_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

OK, INFEASIBLE, E_ARG, E_INVALID_ALLOCATION, E_UNKNOWN_KEY, E_DEGENERATE_PROFILE, E_RANGE = (
    0, 2, 10, 11, 12, 13, 14)


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc -O2 (no fast-math: IEEE FP64)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "cosched_oracle.h"))):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Problem(ctypes.Structure):
    _fields_ = [
        ("n_slots", ctypes.c_int32), ("gpcs_total", ctypes.c_int32), ("n_states", ctypes.c_int32),
        ("state_gpcs", ctypes.c_void_p), ("state_mem", ctypes.c_void_p), ("state_slice", ctypes.c_void_p),
        ("n_slices", ctypes.c_int32), ("n_caps", ctypes.c_int32),
        ("caps_w", ctypes.c_void_p), ("coef_c", ctypes.c_void_p), ("coef_d", ctypes.c_void_p),
        ("objective", ctypes.c_int32), ("alpha", ctypes.c_float),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P = ctypes.POINTER
        L.orc_validate_problem.argtypes = [P(_Problem), ctypes.c_char_p, ctypes.c_int]
        L.orc_validate_features.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                            ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
        L.orc_basis_h.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.orc_basis_j.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.orc_basis_h.restype = None
        L.orc_basis_j.restype = None
        L.orc_rperf.argtypes = [P(_Problem), ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_rperf.restype = ctypes.c_double
        L.orc_eval_set.argtypes = [P(_Problem), ctypes.c_void_p] + [ctypes.c_void_p] * 5
        L.orc_eval_set.restype = None
        L.orc_best_config_members.argtypes = [P(_Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_n_sets.argtypes = [ctypes.c_int64, ctypes.c_int]
        L.orc_n_sets.restype = ctypes.c_int64
        L.orc_unrank.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]
        L.orc_score_range.argtypes = [P(_Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_best_set.argtypes = [P(_Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
        L.orc_exact_allocation.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_greedy_allocation.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_void_p]
        L.orc_greedy_allocation.restype = ctypes.c_int64
        L.orc_hill_climb.argtypes = [P(_Problem), ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.orc_hill_range.argtypes = [P(_Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p]
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class Oracle:
    """Oracle view of one problem (a synth.Problem or anything with its fields)."""

    def __init__(self, pb):
        self.pb = pb
        self._keep = [np.ascontiguousarray(pb.state_gpcs, dtype=np.int32),
                      np.ascontiguousarray(pb.state_mem, dtype=np.int32),
                      np.ascontiguousarray(pb.state_slice, dtype=np.int32),
                      np.ascontiguousarray(pb.caps_w, dtype=np.float32),
                      np.ascontiguousarray(pb.coef_c, dtype=np.float32),
                      np.ascontiguousarray(pb.coef_d, dtype=np.float32)]
        g, m, s, caps, c, d = self._keep
        self.n_slots = int(pb.n_slots)
        self.n_states = int(g.shape[0]) if g.ndim else 0
        self.n_caps = int(caps.shape[0])
        self.n_configs = self.n_states * self.n_caps
        self.st = _Problem(self.n_slots, int(pb.gpcs_total), self.n_states, _ptr(g), _ptr(m), _ptr(s),
                           int(c.shape[1]) if c.ndim == 3 else 0, self.n_caps, _ptr(caps), _ptr(c), _ptr(d),
                           int(pb.objective), float(pb.alpha))

    # -- validation ------------------------------------------------------
    def validate(self) -> Tuple[int, str]:
        msg = ctypes.create_string_buffer(256)
        st = lib().orc_validate_problem(ctypes.byref(self.st), msg, 256)
        return st, msg.value.decode()

    @staticmethod
    def validate_features(F: np.ndarray, jobs: Optional[np.ndarray] = None) -> Tuple[int, str]:
        F = np.ascontiguousarray(F, dtype=np.float32)
        J = None if jobs is None else np.ascontiguousarray(jobs, dtype=np.int32)
        n_jobs = F.shape[0] if J is None else J.shape[0]
        msg = ctypes.create_string_buffer(256)
        st = lib().orc_validate_features(_ptr(F), F.shape[0], _ptr(J), n_jobs, msg, 256)
        return st, msg.value.decode()

    # -- per-set -----------------------------------------------------------
    def _members(self, rows):
        rows = [np.ascontiguousarray(r, dtype=np.float32) for r in rows]
        arr = (ctypes.c_void_p * len(rows))(*[r.ctypes.data for r in rows])
        return arr, rows

    def rperf(self, rows, slot: int, state: int, cap: int) -> float:
        arr, keep = self._members(rows)
        return lib().orc_rperf(ctypes.byref(self.st), arr, slot, state, cap)

    def eval_set(self, rows):
        """Per-config (obj, fair, thr, feasible, rperf[n_cfg][n_slots]) for one set of job rows."""
        arr, keep = self._members(rows)
        n = self.n_configs
        obj, fair, thr = np.zeros(n), np.zeros(n), np.zeros(n)
        feas = np.zeros(n, dtype=np.int32)
        rp = np.zeros((n, self.n_slots))
        lib().orc_eval_set(ctypes.byref(self.st), arr, _ptr(obj), _ptr(fair), _ptr(thr), _ptr(feas), _ptr(rp))
        return obj, fair, thr, feas.astype(bool), rp

    def best_config(self, rows) -> Tuple[int, float]:
        arr, keep = self._members(rows)
        cfg = np.zeros(1, dtype=np.int32)
        obj = np.zeros(1)
        lib().orc_best_config_members(ctypes.byref(self.st), arr, _ptr(cfg), _ptr(obj))
        return int(cfg[0]), float(obj[0])

    def hill_climb(self, rows, start_state: int, start_cap: int) -> Tuple[int, float, int]:
        """(cfg, obj, evals) of the hill climb (reading R22) for one set of job rows."""
        arr, keep = self._members(rows)
        cfg = np.zeros(1, dtype=np.int32)
        obj = np.zeros(1)
        ev = np.zeros(1, dtype=np.int64)
        lib().orc_hill_climb(ctypes.byref(self.st), arr, start_state, start_cap, _ptr(cfg), _ptr(obj), _ptr(ev))
        return int(cfg[0]), float(obj[0]), int(ev[0])

    def hill_range(self, F, start_state: int, start_cap: int, jobs=None, first: int = 0,
                   count: Optional[int] = None):
        """(cfg, obj, evals) arrays of the hill climb for every set of the range."""
        F = np.ascontiguousarray(F, dtype=np.float32)
        J = None if jobs is None else np.ascontiguousarray(jobs, dtype=np.int32)
        n_jobs = F.shape[0] if J is None else J.shape[0]
        if count is None:
            count = n_sets(n_jobs, self.n_slots) - first
        cfg = np.zeros(max(count, 1), dtype=np.int32)
        obj = np.zeros(max(count, 1))
        ev = np.zeros(max(count, 1), dtype=np.int64)
        st = lib().orc_hill_range(ctypes.byref(self.st), _ptr(F), _ptr(J), n_jobs, first, count, start_state,
                                  start_cap, _ptr(cfg), _ptr(obj), _ptr(ev))
        if st:
            raise ValueError(f"oracle hill_range status {st}")
        return cfg[:count], obj[:count], ev[:count]

    # -- queue level ----------------------------------------------------------
    def score_range(self, F, jobs=None, first: int = 0, count: Optional[int] = None):
        F = np.ascontiguousarray(F, dtype=np.float32)
        J = None if jobs is None else np.ascontiguousarray(jobs, dtype=np.int32)
        n_jobs = F.shape[0] if J is None else J.shape[0]
        if count is None:
            count = n_sets(n_jobs, self.n_slots) - first
        cfg = np.zeros(max(count, 1), dtype=np.int32)
        obj = np.zeros(max(count, 1))
        st = lib().orc_score_range(ctypes.byref(self.st), _ptr(F), _ptr(J), n_jobs, first, count,
                                   _ptr(cfg), _ptr(obj))
        if st:
            raise ValueError(f"oracle score_range status {st}")
        return cfg[:count], obj[:count]

    def best_set(self, F, jobs=None, first: int = 0, count: Optional[int] = None):
        F = np.ascontiguousarray(F, dtype=np.float32)
        J = None if jobs is None else np.ascontiguousarray(jobs, dtype=np.int32)
        n_jobs = F.shape[0] if J is None else J.shape[0]
        if count is None:
            count = n_sets(n_jobs, self.n_slots) - first
        sid = np.zeros(1, dtype=np.int64)
        cfg = np.zeros(1, dtype=np.int32)
        obj = np.zeros(1)
        st = lib().orc_best_set(ctypes.byref(self.st), _ptr(F), _ptr(J), n_jobs, first, count,
                                _ptr(sid), _ptr(cfg), _ptr(obj))
        return st, int(sid[0]), int(cfg[0]), float(obj[0])


def n_sets(n_jobs: int, n_slots: int) -> int:
    return int(lib().orc_n_sets(n_jobs, n_slots))


def unrank(n_jobs: int, n_slots: int, set_id: int):
    pos = np.zeros(3, dtype=np.int64)
    st = lib().orc_unrank(n_jobs, n_slots, set_id, _ptr(pos))
    if st:
        raise ValueError("set id out of range")
    return tuple(int(x) for x in pos[:n_slots])


def exact_allocation(n_jobs: int, n_slots: int, set_obj: np.ndarray):
    """(status, best_rank, set_ids in formation order, total, n_matchings)."""
    so = np.ascontiguousarray(set_obj, dtype=np.float64)
    rank = np.zeros(1, dtype=np.int64)
    ids = np.zeros(max(n_jobs // n_slots, 1), dtype=np.int64)
    tot = np.zeros(1)
    nm = np.zeros(1, dtype=np.int64)
    st = lib().orc_exact_allocation(n_jobs, n_slots, _ptr(so), _ptr(rank), _ptr(ids), _ptr(tot), _ptr(nm))
    return st, int(rank[0]), [int(x) for x in ids[: n_jobs // n_slots]], float(tot[0]), int(nm[0])


def greedy_allocation(n_jobs: int, n_slots: int, set_obj: np.ndarray, k: int):
    so = np.ascontiguousarray(set_obj, dtype=np.float64)
    ids = np.zeros(max(k, 1), dtype=np.int64)
    got = lib().orc_greedy_allocation(n_jobs, n_slots, _ptr(so), k, _ptr(ids))
    return [int(x) for x in ids[:got]]


def basis_h(f) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float32)
    h = np.zeros(6)
    lib().orc_basis_h(_ptr(f), _ptr(h))
    return h


def basis_j(f) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float32)
    j = np.zeros(3)
    lib().orc_basis_j(_ptr(f), _ptr(j))
    return j

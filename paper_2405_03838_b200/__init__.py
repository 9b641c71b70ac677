"""B200-native exhaustive, model-driven co-location search (arXiv 2405.03838).

Thin Python binding over libcosched.so (include/cosched.h): the same entry
points, with torch tensors for device memory and streams. Every step of the
search (validation, basis, projection, model evaluation, objective, fairness,
argmax, allocation) runs in the library's sm_100a kernels; this module only
marshals arguments. It never imports the test oracle (oracle/).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import INFEASIBLE, OK, STATUS, Desc, Out

__all__ = ["Scheduler", "CoschedError", "fit", "FitResult", "n_sets", "unrank", "pack_key", "unpack_key", "shard_range_for",
           "get_unique_id", "STATUS"]


class CoschedError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def n_sets(n_jobs: int, n_slots: int) -> int:
    return int(_lib.load().cosched_n_sets(n_jobs, n_slots))


def unrank(n_jobs: int, n_slots: int, set_id: int) -> Tuple[int, ...]:
    pos = (ctypes.c_int64 * 3)()
    st = _lib.load().cosched_unrank(n_jobs, n_slots, set_id, pos)
    if st:
        raise CoschedError(st, "set id out of range")
    return tuple(int(pos[i]) for i in range(n_slots))


def pack_key(obj: float, set_id: int) -> int:
    return int(_lib.load().cosched_pack_key(obj, set_id))


def unpack_key(key: int) -> Tuple[float, int]:
    o = ctypes.c_float()
    s = ctypes.c_int64()
    _lib.load().cosched_unpack_key(key, ctypes.byref(o), ctypes.byref(s))
    return o.value, s.value


def shard_range_for(n_jobs: int, n_slots: int, rank: int, nranks: int) -> Tuple[int, int]:
    a, b = ctypes.c_int64(), ctypes.c_int64()
    st = _lib.load().cosched_shard_range_for(n_jobs, n_slots, rank, nranks, ctypes.byref(a), ctypes.byref(b))
    if st:
        raise CoschedError(st, "bad shard arguments")
    return a.value, b.value


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = _lib.load().cosched_get_unique_id(buf)
    if st:
        raise CoschedError(st, _lib.load().cosched_last_create_error().decode())
    return buf.raw


def _stream_handle(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Scheduler:
    """One search space + model (cosched_desc) bound to one CUDA device.

    `problem` is any object with the cosched_desc fields (e.g. synth.Problem):
    n_slots, gpcs_total, state_gpcs, state_mem, state_slice, caps_w, coef_c,
    coef_d, objective, alpha.
    """

    def __init__(self, problem, device: int = 0):
        L = _lib.load()
        self._keep = [np.ascontiguousarray(problem.state_gpcs, dtype=np.int32),
                      np.ascontiguousarray(problem.state_mem, dtype=np.int32),
                      np.ascontiguousarray(problem.state_slice, dtype=np.int32),
                      np.ascontiguousarray(problem.caps_w, dtype=np.float32),
                      np.ascontiguousarray(problem.coef_c, dtype=np.float32),
                      np.ascontiguousarray(problem.coef_d, dtype=np.float32)]
        g, m, s, caps, c, d = self._keep
        self.n_slots = int(problem.n_slots)
        self.n_states = int(g.shape[0])
        self.n_caps = int(caps.shape[0])
        desc = Desc(self.n_slots, int(problem.gpcs_total), self.n_states, g.ctypes.data, m.ctypes.data,
                    s.ctypes.data, int(c.shape[1]), self.n_caps, caps.ctypes.data, c.ctypes.data, d.ctypes.data,
                    int(problem.objective), float(problem.alpha))
        h = ctypes.c_void_p()
        st = L.cosched_create(ctypes.byref(desc), device, ctypes.byref(h))
        if st:
            raise CoschedError(st, L.cosched_last_create_error().decode())
        self._h = h
        self.device = device
        self._L = L
        self._ws = None
        self._out = None
        self.n_jobs = 0
        self.first, self.count = 0, 0

    def close(self):
        if getattr(self, "_h", None):
            self._L.cosched_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, allow_infeasible: bool = False) -> int:
        if st == OK or (allow_infeasible and st == INFEASIBLE):
            return st
        raise CoschedError(st, self._L.cosched_last_error(self._h).decode())

    # -- multi-GPU ----------------------------------------------------------
    def set_comm(self, uid: Optional[bytes], rank: int, nranks: int):
        buf = None if uid is None else ctypes.create_string_buffer(uid, 128)
        self._check(self._L.cosched_set_comm(self._h, buf, rank, nranks))

    def shard_range(self, n_jobs: int) -> Tuple[int, int]:
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._L.cosched_shard_range(self._h, n_jobs, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def set_shard_view(self, rank: int, nranks: int):
        self._check(self._L.cosched_set_shard_view(self._h, rank, nranks))

    def set_variant(self, variant: int):
        self._check(self._L.cosched_set_variant(self._h, variant))

    def set_search(self, mode: int, start_state: int = 0, start_cap: int = 0):
        """0: exhaustive search (default); 1: hill climbing from (start_state, start_cap)."""
        self._check(self._L.cosched_set_search(self._h, mode, start_state, start_cap))

    def last_search_evals(self) -> int:
        v = ctypes.c_int64()
        self._check(self._L.cosched_last_search_evals(self._h, ctypes.byref(v)))
        return v.value

    def last_timings(self):
        """(prep_ms, score_ms, total_ms) of the last score_all, from CUDA events on its stream."""
        ms = (ctypes.c_float * 3)()
        self._check(self._L.cosched_last_timings(self._h, ms))
        return ms[0], ms[1], ms[2]

    @property
    def greedy_rounds(self) -> int:
        return int(self._L.cosched_last_greedy_rounds(self._h))

    @property
    def last_rescored(self) -> int:
        """Sets of the last score_all re-scored exactly after the tiled scorer (instrumentation)."""
        n = ctypes.c_int64()
        self._check(self._L.cosched_last_rescored(self._h, ctypes.byref(n)))
        return n.value

    @property
    def kernel_launches(self) -> int:
        return int(self._L.cosched_kernel_launches(self._h))

    def workspace_size(self, n_jobs: int) -> int:
        b = ctypes.c_size_t()
        self._check(self._L.cosched_workspace_size(self._h, n_jobs, ctypes.byref(b)))
        return b.value

    # -- the search ------------------------------------------------------------
    def score_all(self, features, jobs=None, with_out: bool = True, stream=None):
        """Score this rank's shard. features: cuda float32 [n_rows][8]; jobs: cuda int32 [n_jobs] or None.
        Returns (obj, cfg) device tensors of the shard (None if with_out=False). Asynchronous."""
        import torch
        assert features.is_cuda and features.dtype == torch.float32 and features.is_contiguous()
        n_rows = features.shape[0]
        if jobs is not None:
            assert jobs.is_cuda and jobs.dtype == torch.int32 and jobs.is_contiguous()
            n_jobs = jobs.shape[0]
        else:
            n_jobs = n_rows
        need = self.workspace_size(n_jobs)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need + 256, dtype=torch.uint8, device=features.device)
        first, count = self.shard_range(n_jobs)
        out_p = None
        if with_out:
            if self._out is None or self._out[0].numel() < count:
                self._out = (torch.empty(max(count, 1), dtype=torch.float32, device=features.device),
                             torch.empty(max(count, 1), dtype=torch.int32, device=features.device))
            out = Out(self._out[0].data_ptr(), self._out[1].data_ptr(), first, count)
            out_p = ctypes.byref(out)
        ws_ptr = self._ws.data_ptr()
        ws_ptr = (ws_ptr + 255) & ~255
        self._check(self._L.cosched_score_all(self._h, features.data_ptr(), n_rows,
                                              None if jobs is None else jobs.data_ptr(), n_jobs, ws_ptr,
                                              self._ws.numel() - (ws_ptr - self._ws.data_ptr()), out_p,
                                              _stream_handle(stream)))
        self.n_jobs = n_jobs
        self.first, self.count = first, count
        if with_out:
            return self._out[0][:count], self._out[1][:count]
        return None, None

    def local_best_key(self) -> int:
        k = ctypes.c_uint64()
        self._check(self._L.cosched_local_best_key(self._h, ctypes.byref(k)))
        return k.value

    def best_set(self):
        """(status, set_id, cfg, obj); collective when a communicator is set."""
        sid, cfg, obj = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_float()
        st = self._check(self._L.cosched_best_set(self._h, ctypes.byref(sid), ctypes.byref(cfg), ctypes.byref(obj)),
                         allow_infeasible=True)
        return st, sid.value, cfg.value, obj.value

    def best_set_begin(self):
        """Enqueue best_set's device work on the last score_all's stream; no synchronisation
        (record an event after it to time the step's device work), then call best_set_end."""
        self._check(self._L.cosched_best_set_begin(self._h))

    def set_timing(self, on: bool):
        """Record the prep / score split events read by last_timings (off by default: they
        cost the scorer's launch its overlap with the gather)."""
        self._check(self._L.cosched_set_timing(self._h, 1 if on else 0))

    def last_step_ms(self) -> float:
        """Device time of the last score_all + best_set (library events around the step's kernels)."""
        ms = ctypes.c_float()
        self._check(self._L.cosched_last_step_ms(self._h, ctypes.byref(ms)))
        return ms.value

    def best_set_end(self):
        """Synchronise and return best_set's (status, set_id, cfg, obj)."""
        sid, cfg, obj = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_float()
        st = self._check(self._L.cosched_best_set_end(self._h, ctypes.byref(sid), ctypes.byref(cfg),
                                                      ctypes.byref(obj)), allow_infeasible=True)
        return st, sid.value, cfg.value, obj.value

    def best_config(self, set_id: int) -> dict:
        cfg, obj, thr, fair = ctypes.c_int32(), ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
        rp = (ctypes.c_float * 3)()
        st = self._check(self._L.cosched_best_config(self._h, set_id, ctypes.byref(cfg), ctypes.byref(obj), rp,
                                                     ctypes.byref(thr), ctypes.byref(fair)), allow_infeasible=True)
        return {"status": st, "cfg": cfg.value, "state": cfg.value // self.n_caps if cfg.value >= 0 else -1,
                "cap": cfg.value % self.n_caps if cfg.value >= 0 else -1, "obj": obj.value,
                "rperf": [rp[i] for i in range(self.n_slots)], "throughput": thr.value, "fairness": fair.value}

    def node_budget(self, set_ids: Sequence[int], gpus_per_node: int, node_power_w: float, objective: int,
                    stream=None):
        """Per-node power caps for the GPUs running set_ids (NEXT #4, reading R23).
        Returns (caps, cfgs, node_obj) host lists."""
        import torch
        n = len(set_ids)
        b = ctypes.c_size_t()
        self._check(self._L.cosched_node_workspace_size(self._h, n, gpus_per_node, float(node_power_w),
                                                        ctypes.byref(b)))
        ws = torch.empty(b.value + 256, dtype=torch.uint8, device=torch.device("cuda", self.device))
        wp = (ws.data_ptr() + 255) & ~255
        ids = (ctypes.c_int64 * n)(*[int(x) for x in set_ids])
        caps = (ctypes.c_int32 * n)()
        cfgs = (ctypes.c_int32 * n)()
        nodes = max(n // max(gpus_per_node, 1), 1)
        obj = (ctypes.c_float * nodes)()
        self._check(self._L.cosched_node_budget(self._h, n, ids, gpus_per_node, float(node_power_w), objective, wp,
                                                b.value, caps, cfgs, obj, _stream_handle(stream)))
        return list(caps), list(cfgs), [obj[i] for i in range(n // gpus_per_node)]

    def evaluate_truth(self, features, truth, jobs=None, stream=None):
        """Worst / proposal / best of the last score_all under a ground-truth model (NEXT #3).
        truth: any object with g_full, n_modules, modules (mapping GPCs -> modules), w_base,
        w_gpc, kappa, f_min, p_max. Returns (prop_obj, prop_fair, best_obj, worst_obj) device
        tensors of the shard and a summary dict (collective with a communicator)."""
        import torch
        dev = features.device
        mods = (ctypes.c_int32 * 17)(*[int(truth.modules.get(g, 0)) for g in range(17)])
        d = _lib.TruthDesc(int(truth.g_full), int(truth.n_modules), mods, float(truth.w_base), float(truth.w_gpc),
                           float(truth.kappa), float(truth.f_min), float(truth.p_max))
        b = ctypes.c_size_t()
        self._check(self._L.cosched_evaluate_workspace_size(self._h, self.n_jobs, ctypes.byref(b)))
        ws = torch.empty(b.value + 256, dtype=torch.uint8, device=dev)
        wp = (ws.data_ptr() + 255) & ~255
        n = max(self.count, 1)
        outs = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(4)]
        o = _lib.EvalOut(*[t.data_ptr() for t in outs])
        sm = _lib.EvalSummary()
        self._check(self._L.cosched_evaluate_truth(self._h, ctypes.byref(d), features.data_ptr(), features.shape[0],
                                                   None if jobs is None else jobs.data_ptr(), wp, b.value,
                                                   ctypes.byref(o), ctypes.byref(sm), _stream_handle(stream)))
        summary = {"n_compared": sm.n_compared, "n_violations": sm.n_violations,
                   "geomean_prop_over_best": sm.geomean_prop_over_best,
                   "geomean_worst_over_best": sm.geomean_worst_over_best}
        return tuple(t[:self.count] for t in outs), summary

    def best_allocation(self, k: int):
        """(status, set_ids, cfgs, total_obj); collective when a communicator is set."""
        ids = (ctypes.c_int64 * max(k, 1))()
        cfgs = (ctypes.c_int32 * max(k, 1))()
        tot = ctypes.c_double()
        nf = ctypes.c_int32()
        st = self._check(self._L.cosched_best_allocation(self._h, k, ids, cfgs, ctypes.byref(tot), ctypes.byref(nf)),
                         allow_infeasible=True)
        n = nf.value
        return st, [ids[i] for i in range(n)], [cfgs[i] for i in range(n)], tot.value


# ---- calibration (include/cosched.h cosched_fit) ----------------

class FitResult:
    """Fitted coefficient table + per-key diagnostics (device tensors unless .cpu() is called)."""

    def __init__(self, coef_c, coef_d, status, count, rms):
        self.coef_c, self.coef_d, self.status, self.count, self.rms = coef_c, coef_d, status, count, rms

    def cpu(self) -> "FitResult":
        return FitResult(*(t.cpu().numpy() for t in (self.coef_c, self.coef_d, self.status, self.count, self.rms)))


def fit(features, n_slices: int, n_caps: int, solo_app, solo_key, solo_rperf, co_app=None, co_partners=None,
        co_key=None, co_rperf=None, stream=None) -> FitResult:
    """Fit C (solo runs) then D (co-run residuals) for every key = cap * n_slices + slice.
    All inputs are cuda tensors (features float32 [n_apps][8]; *_app / *_key / co_partners int32;
    *_rperf float32). Synchronises the stream; raises CoschedError on invalid input."""
    import torch
    dev = features.device
    L = _lib.load()

    def chk(t, dt):
        assert t.is_cuda and t.dtype == dt and t.is_contiguous()
        return t.data_ptr()

    n_co = 0 if co_app is None else int(co_app.shape[0])
    n_part = int(co_partners.shape[1]) if (co_partners is not None and co_partners.dim() == 2) else 1
    d = _lib.FitDesc(n_slices, n_caps, n_part if n_co else 1, features.shape[0], chk(features, torch.float32),
                     solo_app.shape[0], chk(solo_app, torch.int32), chk(solo_key, torch.int32),
                     chk(solo_rperf, torch.float32),
                     n_co, chk(co_app, torch.int32) if n_co else None,
                     chk(co_partners, torch.int32) if n_co else None,
                     chk(co_key, torch.int32) if n_co else None, chk(co_rperf, torch.float32) if n_co else None)
    b = ctypes.c_size_t()
    st = L.cosched_fit_workspace_size(ctypes.byref(d), ctypes.byref(b))
    if st != OK:
        raise CoschedError(st, "cosched_fit_workspace_size")
    ws = torch.empty(b.value + 256, dtype=torch.uint8, device=dev)
    wp = (ws.data_ptr() + 255) & ~255
    nk = n_slices * n_caps
    C = torch.empty((n_caps, n_slices, 6), dtype=torch.float64, device=dev)
    D = torch.empty((n_caps, n_slices, 3), dtype=torch.float64, device=dev)
    status = torch.empty((nk, 2), dtype=torch.int32, device=dev)
    count = torch.empty((nk, 2), dtype=torch.int64, device=dev)
    rms = torch.empty((nk, 2), dtype=torch.float64, device=dev)
    out = _lib.FitOut(C.data_ptr(), D.data_ptr(), status.data_ptr(), count.data_ptr(), rms.data_ptr())
    st = L.cosched_fit(ctypes.byref(d), wp, b.value, ctypes.byref(out), _stream_handle(stream))
    if st != OK:
        raise CoschedError(st, (L.cosched_fit_last_error() or b"").decode())
    return FitResult(C, D, status, count, rms)

#!/usr/bin/env python
"""Benchmark of the exhaustive co-location search (BASELINE.json metric:
candidate configs scored per second, and the fraction of the scorer's roofline).

One step = one pass of the hot path over the queue: validate + basis +
projection + every (set, state, cap) candidate scored + per-set argmax +
per-queue argmax + cross-GPU argmax (cosched_score_all + cosched_best_set).
The greedy job->GPU allocation (cosched_best_allocation) is timed separately
and reported as `allocation_ms`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU, NCCL)

Workload: BASELINE.json config 4 (10,000-job queue, b200 table x 21 caps =
294 configs per pair, 49,995,000 pairs) -- the configuration the 1/2/4/8-GPU
metric is quoted on; synthetic class-shaped inputs (synth/).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample.
"""
from __future__ import annotations

import argparse
import copy
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "candidate configs scored/sec (1/2/4/8 B200) and % of FP32/HBM roofline"
UNIT = "candidates/s"
# Roofline of the set scorer (DESIGN.md §5 "Roofline"). `roofline` follows the
# contract: SURVEY.md §8(d)'s algorithmic FP32 operations per candidate (the
# method's cheapest exact form: pair P2 = 3 FADD + 1 FMUL + 1 FMNMX + 2 FSETP = 7,
# P1 = 6; triple P2 = 10, P1 = 9; solo P2 = 3, P1 = 2) against the FP32 lane peak
# 148 SM x 128 lanes x clock. `roofline_strict` is this implementation's own
# binding unit: the ALU pipe (FMNMX3: 64 lanes/clk/SM, profiles/r01/
# microbench_pipes*) with >= 1.5 ALU lane-ops per pair candidate (one 3-input min
# for the masked Fairness test, half a 3-input max for the argmax), 2.5 per triple.
FP32_OPS_PER_CAND = {(1, 1): 2, (1, 2): 3, (2, 1): 6, (2, 2): 7, (3, 1): 9, (3, 2): 10}
FP32_LANES_PER_SM_CLK = 128
ALU_OPS_PER_CAND = {1: 1.0, 2: 1.5, 3: 2.5}
ALU_LANES_PER_SM_CLK = 64
N_SM = 148


def _ncu_summary(workload: str):
    """The committed ncu --set full summary of the scorer
    (profiles/<round>/<workload>_scorer_ncu_summary.json), or (None, None)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"{workload.lower()}_scorer_ncu_summary.json")),
                       reverse=True):
        try:
            with open(path) as f:
                return json.load(f), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def _traffic(workload: str, n_slots: int):
    """DRAM bytes per scorer launch from the committed ncu --set full capture, or None."""
    d, src = _ncu_summary(workload)
    try:
        return float(d["traffic_bytes_per_launch"]) / 1e9, src
    except Exception:
        return None, None


def _ncu_pipes(workload: str):
    """Issue and pipe utilisation of the scorer from the committed ncu capture (SURVEY 8(d):
    report pipe utilisation and the FMA-FLOP/s against 148 x 128 x 2 x clock)."""
    d, src = _ncu_summary(workload)
    if not d:
        return None
    keys = {"issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "fmaheavy_pipe_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"}
    out = {}
    for k, m in keys.items():
        try:
            out[k] = float(d[m])
        except Exception:
            pass
    out["source"] = src
    return out


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled every
    2 ms from a thread (the timed region of C4 is ~35 ms, shorter than nvidia-smi's
    100 ms loop), with nvidia-smi as the fallback when NVML is unavailable."""

    # NVML clocks-event reason bits (nvml.h nvmlClocksEventReason*)
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reason bits) from NVML
        self.power = []    # W, NVML
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self._stop.is_set():
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx,
                                             int(get_reasons(h))))
                        try:
                            self.power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
                        except Exception:
                            pass
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 2.0:  # live before the timed region starts
                time.sleep(0.001)
            return self
        except Exception:
            self.samples = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.t:
            self.t.join(timeout=1.0)

    def summary(self):
        if self.samples:
            sm = [s[0] for s in self.samples]
            reasons = sorted({name for _, _, bits in self.samples for bit, name in self.REASONS.items() if bits & bit})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                    "reasons": reasons, "samples": len(sm),
                    "power_w": statistics.median(self.power) if self.power else None,
                    "source": "NVML, 2 ms polling during the timed steps"}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 100"}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_rate(pb, F, n_slots, budget_s=12.0, first=0):
    """Oracle (as it stands, single-threaded FP64) on all host cores: disjoint set chunks,
    one process per core, sized from a short calibration so the run takes ~budget_s."""
    import multiprocessing as mproc

    import oracle
    o = oracle.Oracle(pb)
    n_jobs = F.shape[0]
    total = oracle.n_sets(n_jobs, n_slots)
    t0 = time.perf_counter()
    probe = min(2000, total)
    o.score_range(F, None, first, probe)
    per_set = (time.perf_counter() - t0) / max(probe, 1)
    cores = os.cpu_count() or 1
    chunk = max(1, min(total // cores, int(budget_s / max(per_set, 1e-9))))
    ctx = mproc.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        starts = [(first + i * chunk) % max(total - chunk, 1) for i in range(cores)]
        pool.starmap(_oracle_chunk, [(pb, F, s, chunk) for s in starts])
    dt = time.perf_counter() - t0
    n_cand = cores * chunk * pb.n_configs
    return {"value": n_cand / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"{cores} processes x {chunk} consecutive sets ({cores * chunk} sets, "
                      f"{n_cand:.3g} candidates) of {pb.name} with {n_jobs} jobs, single-threaded FP64 "
                      f"un-factorised oracle per process, {dt:.1f} s wall"}


def _oracle_chunk(pb, F, start, count):
    import oracle
    oracle.Oracle(pb).score_range(F, None, start, count)
    return count


def run_reference(args):
    """--impl reference: the CPU oracle (the paper's method written out plainly) on host cores."""
    world, rank, local = _dist_env()
    if rank != 0:
        return 0
    from synth import bench_config
    pb, F = bench_config(args.config)
    n_slots = pb.n_slots
    # bounded sample per step, sized so the whole run stays within a few minutes;
    # warm-up steps are short untimed samples (process start-up, page-in)
    for k in range(args.warmup):
        cpu_oracle_rate(pb, F, n_slots, budget_s=0.5, first=k * 104729)
    steps = []
    info = None
    step_ms = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        info = cpu_oracle_rate(pb, F, n_slots, budget_s=args.ref_budget, first=k * 7919)
        step_ms.append((time.perf_counter() - t0) * 1e3)
        steps.append(info["value"])
    value = statistics.median(steps)
    import oracle
    n_cand_step = oracle.n_sets(int(F.shape[0]), n_slots) * pb.n_configs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # a step is one bounded sample of the workload (its wall time, measured);
            # the whole workload at the sampled rate is reported separately
            "ms_per_step": statistics.median(step_ms),
            "ms_per_workload_extrapolated": n_cand_step / value * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n_jobs": int(F.shape[0]), "n_slots": n_slots,
                       "n_configs": pb.n_configs, "table": pb.name, "objective": pb.objective,
                       "alpha": pb.alpha, "parallelism": "host processes"},
            "cpu_baseline": {"kind": info["kind"], "cores": info["cores"], "cpu_model": info.get("cpu_model"),
                             "sample": info["sample"], "value": value, "unit": UNIT},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def calibration_metrics(pb, F, dev, args):
    """Time cosched_fit on a training set for the bench queue:
    every app solo on every (slice, cap) key plus --calib-coruns co-runs, measured on the
    synthetic GPU (synth/ground_truth.py, sigma = 0.01 noise). Device time, CUDA events."""
    import torch

    import paper_2405_03838_b200 as cs
    from synth.ground_truth import make_training_set

    ts = make_training_set(F, pb, n_corun=args.calib_coruns, seed=3000, noise=0.01)
    d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
    targs = (d(F, np.float32), pb.n_slices, pb.n_caps, d(ts.solo_app, np.int32), d(ts.solo_key, np.int32),
             d(ts.solo_rperf, np.float32), d(ts.co_app, np.int32), d(ts.co_partners, np.int32),
             d(ts.co_key, np.int32), d(ts.co_rperf, np.float32))
    for _ in range(2):
        r = cs.fit(*targs)
    times = []
    stream = torch.cuda.current_stream()
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = cs.fit(*targs)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    st = r.status.cpu().numpy()
    # the paper's workflow on the fitted table (NEXT #3): search the queue, evaluate the
    # proposals against the ground truth (worst / proposal / best geometric means)
    from synth.ground_truth import B200 as truth
    pbf = copy.copy(pb)
    pbf.coef_c = r.coef_c.cpu().numpy().astype(np.float32)
    pbf.coef_d = r.coef_d.cpu().numpy().astype(np.float32)
    sf = cs.Scheduler(pbf, device=dev.index or 0)
    Fd = targs[0]
    sf.score_all(Fd)
    sf.evaluate_truth(Fd, truth)  # warm: output buffers, lazy module load
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, summ = sf.evaluate_truth(Fd, truth)
    e1.record(stream)
    torch.cuda.synchronize()
    pipeline = dict(summ)
    pipeline["evaluate_ms"] = e0.elapsed_time(e1)
    pipeline["note"] = ("C, D fitted on the synthetic GPU; the fitted table searched over the queue; proposals "
                        "scored by the ground truth (PAPER.md L752/L777 analogue)")
    # hill climbing (NEXT #2) on the calibrated table: its decisions against the
    # exhaustive search on the same table, and its proposals scored by the ground truth
    obj_e, cfg_e = sf.score_all(Fd)
    obj_e, cfg_e = obj_e.clone(), cfg_e.clone()
    hill = {}
    balanced = int(np.argmin(np.asarray(pb.state_gpcs).max(axis=1)))
    for name, start in (("first_state_pmax", (0, pb.n_caps - 1)), ("balanced_pmax", (balanced, pb.n_caps - 1))):
        sf.set_search(1, *start)
        obj_h, cfg_h = sf.score_all(Fd)
        evals = sf.last_search_evals()
        feas = (cfg_e >= 0) & (cfg_h >= 0)
        ratio = obj_h[feas].double() / obj_e[feas].double()
        _, hs = sf.evaluate_truth(Fd, truth)
        hill[name] = {"same_config_as_exhaustive": float((cfg_h == cfg_e).double().mean().item()),
                      "objective_ratio_geomean": float(torch.exp(torch.log(ratio).mean()).item()) if ratio.numel() else None,
                      "evals_per_set": evals / max(cfg_e.numel(), 1),
                      "truth_geomean_prop_over_best": hs["geomean_prop_over_best"]}
        sf.set_search(0)
    pipeline["hill_climb_on_calibrated_table"] = hill
    sf.close()
    n_solo, n_co = len(ts.solo_app), len(ts.co_app)
    npart = ts.co_partners.shape[1] if n_co else 0
    # algorithmic bytes: each sample record once (app, key, rperf, partners) + each app's counters
    algo = n_solo * 12 + n_co * (12 + 4 * npart) + F.shape[0] * 32
    peaks, src = _peaks()
    gbs = algo / (ms * 1e-3) / 1e9
    return {"workload": f"{args.config} queue: every app solo on every (slice, cap) key + "
                        f"{args.calib_coruns} co-runs, synthetic GPU, sigma 0.01",
            "n_apps": int(F.shape[0]), "n_keys": int(pb.n_slices * pb.n_caps), "solo_samples": n_solo,
            "corun_samples": n_co, "ms": ms, "samples_per_s": (n_solo + n_co) / (ms * 1e-3),
            "keys_fitted": [int((st[:, 0] == 0).sum()), int((st[:, 1] == 0).sum())],
            "algorithmic_bytes": algo, "achieved_gbs": gbs, "hbm_peak_gbs": peaks.get("hbm_gbs"),
            "hbm_frac": gbs / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None, "peak_source": src,
            "pipeline": pipeline}


def hill_metrics(sched, Fd, pb, stream, args):
    """Hill climbing (cosched_set_search mode 1, NEXT #2) over the same queue: device time,
    evaluations, and decision quality against the exhaustive search just timed."""
    import torch
    obj_e, cfg_e = sched.score_all(Fd, None, with_out=True, stream=stream)
    obj_e, cfg_e = obj_e.clone(), cfg_e.clone()

    def climb(start):
        sched.set_search(1, *start)
        times = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            obj_h, cfg_h = sched.score_all(Fd, None, with_out=True, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        evals = sched.last_search_evals()
        feas = (cfg_e >= 0) & (cfg_h >= 0)
        ratio = (obj_h[feas].double() / obj_e[feas].double())
        return {"start": {"state": int(start[0]), "cap": int(start[1])}, "ms": min(times), "sets": int(cfg_e.numel()),
                "evals": int(evals), "evals_per_set": evals / max(cfg_e.numel(), 1),
                "evals_per_s": evals / (min(times) * 1e-3),
                "same_config_as_exhaustive": float((cfg_h == cfg_e).double().mean().item()),
                "objective_ratio_mean": float(ratio.mean().item()) if ratio.numel() else None,
                "objective_ratio_geomean": float(torch.exp(torch.log(ratio).mean()).item()) if ratio.numel() else None}

    # the first state of the table at P_max, and the most even split (the first
    # state with the smallest largest slot, shared memory) at P_max
    out = climb((0, pb.n_caps - 1))
    balanced = int(np.argmin(np.asarray(pb.state_gpcs).max(axis=1)))
    out["balanced_start"] = climb((balanced, pb.n_caps - 1))
    sched.set_search(0)
    return out


def shard_projection(sched, Fd, stream, t1_ms, cand_per_step, args):
    """Strong-scaling projection on ONE GPU: every rank's shard of a W-way run
    (cosched_set_shard_view, the same set ranges cosched_shard_range gives rank r
    of W) timed alone as a full step (validate + project + gather + score + local
    best), L2 flushed between steps. The W-GPU step is bounded below by the
    slowest shard; the NCCL u64 max all-reduce (~10-30 us over NVLink, SURVEY
    8(e)) is not included. A projection, not a multi-GPU measurement."""
    import torch

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=Fd.device)
    out = {"method": "each rank's shard timed alone on one GPU (fake-rank view), max over ranks; "
                     "excludes the NCCL all-reduce", "t1_ms": t1_ms, "per_w": {}}
    for W in args.shard_ws:
        per_rank, prep, score = [], [], []
        for r in range(W):
            sched.set_shard_view(r, W)
            for _ in range(2):
                sched.score_all(Fd, None, with_out=True, stream=stream)
                sched.best_set()
            ts, ps, ss = [], [], []
            for k in range(args.shard_steps):
                flush.fill_(k & 0xFF)
                sched.score_all(Fd, None, with_out=True, stream=stream)
                sched.best_set()
                ts.append(sched.last_step_ms())
            sched.set_timing(True)  # the prep / score split: a second pass (its events cost the PDL overlap)
            for k in range(args.shard_steps):
                flush.fill_(k & 0xFF)
                sched.score_all(Fd, None, with_out=True, stream=stream)
                sched.best_set()
                p_, s_, _ = sched.last_timings()
                ps.append(p_)
                ss.append(s_)
            sched.set_timing(False)
            per_rank.append(statistics.median(ts))
            prep.append(statistics.median(ps))
            score.append(statistics.median(ss))
        sched.set_shard_view(0, 1)
        tmax = max(per_rank)
        out["per_w"][str(W)] = {"max_ms": tmax, "min_ms": min(per_rank), "per_rank_ms": per_rank, "prep_ms": prep, "score_ms": score,
                                "projected_speedup": t1_ms / tmax,
                                "projected_candidates_per_s": cand_per_step / (tmax * 1e-3)}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2405_03838_b200 as cs
    from synth import bench_config

    world, rank, local = _dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pb, F = bench_config(args.config)
    n_jobs = F.shape[0]
    sched = cs.Scheduler(pb, device=local)
    if args.variant is not None:
        sched.set_variant(args.variant)
    if world > 1:
        uid = [cs.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        sched.set_comm(uid[0], rank, world)
    stream = torch.cuda.current_stream()
    Fd = torch.from_numpy(F).to(dev)
    first, count = sched.shard_range(n_jobs)
    n_cfg = pb.n_configs
    total_sets = cs.n_sets(n_jobs, pb.n_slots)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        sched.score_all(Fd, None, with_out=True, stream=stream)
        return sched.best_set()

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    score_ms, prep_ms, lib_ms = [], [], []
    launches0 = sched.kernel_launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # evict L2 between timed steps (not timed)
            e0, e1 = ev[k]
            e0.record(stream)
            sched.score_all(Fd, None, with_out=True, stream=stream)
            sched.best_set_begin()
            e1.record(stream)  # after the step's last device work (the result is in pinned host memory)
            res = sched.best_set_end()
            lib_ms.append(sched.last_step_ms())
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = sched.kernel_launches - launches0
    # the prep / scorer split (roofline kernel time) from a second, untimed pass
    # with the split events on: they cost the scorer's launch its PDL overlap
    # with the gather, so the timed steps above run without them
    sched.set_timing(True)
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        sched.score_all(Fd, None, with_out=True, stream=stream)
        sched.best_set()
        p, s, _ = sched.last_timings()
        prep_ms.append(p)
        score_ms.append(s)
    sched.set_timing(False)
    torch.cuda.synchronize()
    outer_ms = [a.elapsed_time(b) for a, b in ev]
    # a step's device time: the library's events on the launching stream, recorded
    # before its first kernel and after its last (cosched_last_step_ms) -- the
    # outer torch events also hold the host's Python -> C call latency before the
    # first launch (reported as ms_per_step_outer_events). The step time is the
    # median over the timed steps, max over ranks
    step_ms = lib_ms
    t_local = statistics.median(step_ms)
    if world > 1:
        t = torch.tensor([t_local, sum(step_ms), statistics.median(score_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_per_step, t_total, score_med = float(t[0].item()), float(t[1].item()), float(t[2].item())
    else:
        ms_per_step, t_total, score_med = t_local, sum(step_ms), statistics.median(score_ms)
    ms_per_step_mean = t_total / args.steps
    cand_per_step = total_sets * n_cfg
    value = cand_per_step / (ms_per_step * 1e-3)

    # end to end through the public API with host buffers: pinned H2D of the
    # features, the search, D2H of the result (best set id/cfg/obj) every step
    Fh = torch.from_numpy(F).pin_memory()
    e2e_times = []
    for k in range(max(2, args.steps)):
        flush.fill_((k + 1) & 0xFF)  # L2 evicted between e2e steps too (not timed)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        Fd.copy_(Fh, non_blocking=True)
        r = step()
        e2e_times.append(time.perf_counter() - t0)
    e2e_t = statistics.median(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())

    # allocation latency (timed separately)
    alloc_ms = None
    alloc_rounds = None
    node_info = None
    if args.alloc_k:
        sched.score_all(Fd, None, with_out=True, stream=stream)
        torch.cuda.synchronize()
        # one untimed allocation (first-call setup), then the median of 3 (host wall
        # clock: the allocation synchronises with the host between its batches)
        sched.best_allocation(args.alloc_k)
        alloc_times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, ids, cfgs, tot = sched.best_allocation(args.alloc_k)
            alloc_times.append((time.perf_counter() - t0) * 1e3)
        alloc_ms = statistics.median(alloc_times)
        alloc_rounds = sched.greedy_rounds
        # node-level power budgeting of the allocation (NEXT #4): nodes of 8 GPUs under
        # a budget of 6 kW (75 % of 8 x P_max), caps per GPU by the exact knapsack DP
        node_info = None
        G = 8
        if pb.n_slots >= 2 and len(ids) >= G:
            use = ids[:len(ids) // G * G]
            node_w = 0.75 * G * float(max(pb.caps_w))
            sched.node_budget(use, G, node_w, pb.objective)  # warm
            t1 = time.perf_counter()
            caps_n, cfgs_n, nobj = sched.node_budget(use, G, node_w, pb.objective)
            node_ms = (time.perf_counter() - t1) * 1e3
            fin = [v for v in nobj if v > -math.inf]
            node_info = {"nodes": len(nobj), "gpus_per_node": G, "node_budget_w": node_w, "ms": node_ms,
                         "feasible_nodes": len(fin), "mean_node_objective": (sum(fin) / len(fin)) if fin else None,
                         "mean_gpu_cap_w": float(np.mean([float(pb.caps_w[c]) for c in caps_n if c >= 0]))}

    if rank == 0:
        peaks, peak_src = _peaks()
        sm_clk = peaks.get("sm_max_mhz", 1965.0)
        alu_peak = N_SM * ALU_LANES_PER_SM_CLK * sm_clk * 1e6 / 1e12  # T lane-ops/s
        fp32_peak = N_SM * FP32_LANES_PER_SM_CLK * sm_clk * 1e6 / 1e12
        score_avg_ms = score_med  # the scorer's median per step (CUDA events on the launching stream)
        local_cand = count * n_cfg  # per-rank candidates of one scorer launch (rank 0's shard)
        ops = FP32_OPS_PER_CAND[(pb.n_slots, pb.objective)]
        alu_ops = ALU_OPS_PER_CAND[pb.n_slots]
        traffic_gb, traffic_src = _traffic(args.config, pb.n_slots)
        cand_rate = local_cand / (score_avg_ms * 1e-3)
        achieved = cand_rate * ops / 1e12
        achieved_alu = cand_rate * alu_ops / 1e12
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "ms_per_step_mean": ms_per_step_mean,
            "ms_per_step_outer_events": statistics.median(outer_ms),
            "step_timing": "median over steps of the device time between the library's events before the step's "
                           "first kernel and after its last (cosched_last_step_ms), max over ranks; "
                           "ms_per_step_outer_events: torch events around the API calls (adds host call latency)",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "n_jobs": n_jobs, "n_slots": pb.n_slots,
                       "n_sets": total_sets, "n_configs": n_cfg, "candidates_per_step": cand_per_step,
                       "table": pb.name, "objective": pb.objective, "alpha": pb.alpha,
                       "parallelism": f"set-range shards x{world}, NCCL u64-max argmax",
                       "l2": "flushed between timed steps (256 MB write)",
                       "scorer": "fast" if (args.variant is None or args.variant == 1) else "generic"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": fp32_peak, "unit": "T FP32 lane-ops/s",
                         "frac": achieved / fp32_peak, "traffic": traffic_gb, "traffic_unit": "GB per launch",
                         "traffic_source": traffic_src, "traffic_measured_in_this_run": False,
                         "algorithmic_bytes_per_launch_gb": count * 8 / 1e9,
                         "kernel": "set scorer", "ops_per_candidate": ops,
                         "ops_source": "SURVEY.md 8(d) algorithmic FP32 ops per candidate",
                         "kernel_ms": score_avg_ms, "kernel_share_of_step": score_avg_ms / ms_per_step,
                         "peak_source": f"148 SM x 128 FP32 lanes x sm_max_mhz ({peak_src} MEASURED_PEAKS.json)",
                         "ncu_pipes": _ncu_pipes(args.config)},
            "roofline_strict": {"bound": "alu", "achieved": achieved_alu, "peak": alu_peak, "unit": "T ALU lane-ops/s",
                                "frac": achieved_alu / alu_peak, "ops_per_candidate": alu_ops,
                                "ops_source": "ALU-pipe ops the exact method needs per candidate (FMNMX3)",
                                "peak_source": f"148 SM x 64 ALU lanes x sm_max_mhz ({peak_src} MEASURED_PEAKS.json)"},
            "e2e": {"value": cand_per_step / e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(F.nbytes),
                    "d2h_bytes_per_step": 8 + 32},
            "gpu_launches": int(launches),
            "rescored_sets": sched.last_rescored,
            "prep_ms": statistics.mean(prep_ms), "allocation_ms": alloc_ms, "allocation_k": args.alloc_k, "allocation_rounds": alloc_rounds,
            "node_budget": node_info,
            "clocks": clocks,
        }
        # the paper's own selection-quality numbers, quoted with their hardware
        # (context only, not comparable: A100 measurements of 18 real pairs)
        line["paper_context"] = {
            "hardware": "NVIDIA A100 40GB PCIe, Threadripper PRO 3955WX, CUDA 11.5 (PAPER.md L503-519)",
            "problem1_geomean_weighted_speedup_proposal_vs_best": [1.52, 1.54],
            "problem1_setting": "P = 230 W, alpha = 0.2, 18 pairs (PAPER.md L754, 5.2.2)",
            "model_mean_abs_rel_error_throughput_fairness": [0.097, 0.145],
            "model_error_source": "PAPER.md L742 (5.2.1)",
            "fairness_violations": 0,
            "our_analogue": "calibration.pipeline: geomean proposal/best on the synthetic-GPU ground truth"}
        if args.shard_ws and world == 1:
            line["shard_projection"] = shard_projection(sched, Fd, stream, ms_per_step, cand_per_step, args)
        if args.hill:
            line["hill_climb"] = hill_metrics(sched, Fd, pb, stream, args)
        if args.calib_coruns > 0:
            line["calibration"] = calibration_metrics(pb, F, dev, args)
        if args.cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_oracle_rate(pb, F, pb.n_slots, budget_s=args.ref_budget)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", type=int, default=None, help="pair scorer: 1 fast (default), 0 generic")
    ap.add_argument("--alloc-k", type=int, default=5000)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-hill", dest="hill", action="store_false", help="skip the hill-climbing measurement")
    ap.add_argument("--calib-coruns", type=int, default=1000000,
                    help="co-runs of the calibration timing (0: skip the calibration measurement)")
    ap.add_argument("--ref-budget", type=float, default=10.0, help="seconds of oracle work per reference step")
    ap.add_argument("--shard-ws", type=lambda s: [int(x) for x in s.split(",") if x], default=[2, 4, 8],
                    help="W values of the one-GPU strong-scaling projection (empty: skip)")
    ap.add_argument("--shard-steps", type=int, default=5)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        args.ref_budget = min(args.ref_budget, 150.0 / max(args.steps, 1))
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

"""The oracle (as it stands: single-threaded FP64, tests only) over every host core:
disjoint consecutive set-id chunks, one forked process per core, results
gathered in colex order. No arithmetic here -- only the work split."""
from __future__ import annotations

import multiprocessing as mproc
import os

import numpy as np

_JOB = {}


def _chunk(args):
    first, count = args
    import oracle
    cfg, obj = oracle.Oracle(_JOB["pb"]).score_range(_JOB["F"], _JOB["jobs"], first, count)
    return first, cfg, obj


def score_range_all_cores(pb, F, jobs=None, first=0, count=None, procs=None):
    """(cfg int32[count], obj float64[count], cores) of sets [first, first+count) by the oracle."""
    import oracle
    n = F.shape[0] if jobs is None else len(jobs)
    total = oracle.n_sets(n, pb.n_slots)
    count = total - first if count is None else count
    procs = procs or os.cpu_count() or 1
    n_chunks = max(1, min(count, procs * 8))  # several chunks per core: even finish
    bounds = np.linspace(first, first + count, n_chunks + 1).astype(np.int64)
    _JOB.update(pb=pb, F=F, jobs=jobs)
    cfg = np.empty(count, np.int32)
    obj = np.empty(count, np.float64)
    ctx = mproc.get_context("fork")
    with ctx.Pool(procs) as pool:
        for f0, c, o in pool.imap_unordered(_chunk, [(int(a), int(b - a)) for a, b in zip(bounds[:-1], bounds[1:])]):
            cfg[f0 - first:f0 - first + len(c)] = c
            obj[f0 - first:f0 - first + len(o)] = o
    return cfg, obj, procs

"""Per-rank scorer time of W-way pair shards on one GPU (fake-rank views), against the
shard's tile count, for calibrating the shard DP's time model (api.cu pair_block_bounds).
usage: python tools/shard_prof.py C4 2 3 4 5 6 7 8 10 12 16   (W:r = only rank r of W)"""
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs  # noqa: E402
from synth import bench_config  # noqa: E402

cfgname = sys.argv[1]
specs = sys.argv[2:] or ['8']
pb, F = bench_config(cfgname)
s = cs.Scheduler(pb)
Fd = torch.from_numpy(F).cuda()
st = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
cur = torch.cuda.current_stream()
N = F.shape[0]


def col_at(v):
    lo, hi = 0, N
    while lo < hi:
        m = (lo + hi) // 2
        if m * (m - 1) // 2 >= v:
            hi = m
        else:
            lo = m + 1
    return lo


for spec in specs:
    W = int(spec.split(':')[0])
    for r in ([int(spec.split(':')[1])] if ':' in spec else range(W)):
        s.set_shard_view(r, W)
        first, count = s.shard_range(N)
        c0, c1 = col_at(first), col_at(first + count)
        B0, B1 = (c0 + 63) // 64, (c1 + 63) // 64
        tiles = B1 * (B1 + 1) // 2 - B0 * (B0 + 1) // 2
        for _ in range(2):
            s.score_all(Fd, None, with_out=True, stream=st)
            s.best_set()
        ts, ss, ps = [], [], []
        for k in range(7):
            with torch.cuda.stream(st):  # the flush on the step's stream: it must not overlap the step
                flush.fill_(k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s.score_all(Fd, None, with_out=True, stream=st)
            s.best_set_begin()
            e1.record(st)
            s.best_set_end()
            ts.append(s.last_step_ms())
        s.set_timing(True)  # the prep / score split: a second pass (its events cost the PDL overlap)
        for k in range(7):
            with torch.cuda.stream(st):
                flush.fill_(k)
            s.score_all(Fd, None, with_out=True, stream=st)
            s.best_set()
            p_, s_, _ = s.last_timings()
            ps.append(p_)
            ss.append(s_)
        s.set_timing(False)
        print(f"W={W} r={r} blocks=[{B0},{B1}) tiles={tiles} rounds={tiles / 296:.3f} R={tiles % 296} "
              f"step={statistics.median(ts):.4f} prep={statistics.median(ps):.4f} score={statistics.median(ss):.4f}",
              flush=True)
s.set_shard_view(0, 1)

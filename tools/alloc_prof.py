"""Run one greedy allocation of a bench config (for ncu launch lists / timing breakdowns).
usage: python tools/alloc_prof.py C5 666"""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs  # noqa: E402
from synth import bench_config  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
pb, F = bench_config(cfgname)
s = cs.Scheduler(pb)
Fd = torch.from_numpy(F).cuda()
s.score_all(Fd)
torch.cuda.synchronize()
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
times = []
for rep in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, ids, cfgs, tot = s.best_allocation(k)
    torch.cuda.synchronize()
    times.append(1e3 * (time.perf_counter() - t0))
    print(f"allocation {cfgname} k={k}: {times[-1]:.2f} ms, rounds {s.greedy_rounds}, found {len(ids)}", flush=True)
if reps > 2:
    import statistics
    print(f"allocation {cfgname} k={k}: median of the last {reps - 1}: {statistics.median(times[1:]):.2f} ms", flush=True)

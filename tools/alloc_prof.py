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
for rep in range(2):
    t0 = time.perf_counter()
    st, ids, cfgs, tot = s.best_allocation(k)
    torch.cuda.synchronize()
    print(f"allocation {cfgname} k={k}: {1e3 * (time.perf_counter() - t0):.2f} ms, rounds {s.greedy_rounds}, "
          f"found {len(ids)}", flush=True)

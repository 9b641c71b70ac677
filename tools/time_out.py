"""Scorer time with and without the per-set outputs (obj/cfg stores), C4."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs
from synth import bench_config
pb, F = bench_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
s = cs.Scheduler(pb)
s.set_timing(True)
Fd = torch.from_numpy(F).cuda()
for with_out in (True, False, True, False):
    for _ in range(3):
        s.score_all(Fd, with_out=with_out)
    ts = []
    for _ in range(5):
        s.score_all(Fd, with_out=with_out)
        ts.append(s.last_timings()[1])
    print(f"with_out={with_out}: scorer {min(ts):.3f} ms (median {sorted(ts)[2]:.3f})")

"""Time cosched_evaluate_truth on a bench queue (warm), exhaustive proposals."""
import sys
import time
import torch
sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs
from synth import bench_config
from synth.ground_truth import B200
pb, F = bench_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
s = cs.Scheduler(pb)
Fd = torch.from_numpy(F).cuda()
s.score_all(Fd)
for rep in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, sm = s.evaluate_truth(Fd, B200)
    e1.record()
    torch.cuda.synchronize()
    print(f"evaluate_truth: {e0.elapsed_time(e1):.2f} ms  {sm['geomean_prop_over_best']:.6f}")

import sys, torch
sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs
from synth import bench_config
pb, F = bench_config("C4")
s = cs.Scheduler(pb)
Fd = torch.from_numpy(F).cuda()
s.score_all(Fd); torch.cuda.synchronize()
s.best_allocation(5000); torch.cuda.synchronize()

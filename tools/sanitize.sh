#!/bin/bash
# compute-sanitizer passes over small problems that touch every kernel
# (memcheck: out-of-bounds / misaligned; racecheck + synccheck: shared-memory hazards in the tiled scorers).
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
cat > /tmp/san_case.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_03838_b200 as cs
from synth import make_features, make_problem, bench_config
from synth.ground_truth import B200, make_training_set
for table, n in (("b200", 130), ("b200_3way", 40)):
    pb = make_problem(table, "c10", coef_seed=5, alpha=0.2)
    F, _ = make_features(n, seed=5)
    s = cs.Scheduler(pb)
    Fd = torch.from_numpy(F).cuda()
    s.score_all(Fd); s.best_set(); s.best_allocation(n // pb.n_slots // 2)
    s.evaluate_truth(Fd, B200)
    ids = list(range(8))
    s.node_budget(ids, 4, 3000.0, 2)
    s.set_search(1, 0, 0); s.score_all(Fd); s.best_set()
    s.set_variant(0); s.set_search(0); s.score_all(Fd)
    s.set_variant(1)
    for r in range(3):  # fake-rank shards: partial boundary column blocks, row-sharded gather
        s.set_shard_view(r, 3); s.score_all(Fd); s.best_set()
    s.set_shard_view(0, 1)
pb, F = bench_config("C2")
ts = make_training_set(F, pb, n_corun=100, seed=1)
d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()
cs.fit(d(F, np.float32), pb.n_slices, pb.n_caps, d(ts.solo_app, np.int32), d(ts.solo_key, np.int32),
       d(ts.solo_rperf, np.float32), d(ts.co_app, np.int32), d(ts.co_partners, np.int32), d(ts.co_key, np.int32),
       d(ts.co_rperf, np.float32))
s = cs.Scheduler(pb); s.score_all(d(F, np.float32)); s.best_allocation(4)
torch.cuda.synchronize()
print("case done")
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python /tmp/san_case.py > $OUT/$tool.txt 2>&1
  echo "$tool rc=$?: $(tail -2 $OUT/$tool.txt | tr '\n' ' ')"
done

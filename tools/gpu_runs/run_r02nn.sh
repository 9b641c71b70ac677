mkdir -p gpurun_out/r02nn
O=gpurun_out/r02nn
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
bash tools/gpu_bench_profile.sh r02nn_c4 > $O/prof.log 2>&1
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 666 > $O/bench_c5.json 2> $O/bench_c5.err
tail -2 $O/pytest.txt; tail -1 $O/smoke.txt
python -c "
import json
for f in ['gpurun_out/r02nn_c4/bench.json','$O/bench_c5.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], d['prep_ms'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['allocation_ms'], {w:round(v['projected_speedup'],3) for w,v in d['shard_projection']['per_w'].items()})
"

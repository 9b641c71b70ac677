mkdir -p gpurun_out/r02w
O=gpurun_out/r02w
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
tail -n 2 $O/pytest.txt
python -c "
import json
d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ms_per_step_outer_events'], d['prep_ms'], d['roofline']['frac'], d['allocation_ms'], {w:round(v['projected_speedup'],3) for w,v in d['shard_projection']['per_w'].items()})
"

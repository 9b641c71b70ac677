mkdir -p gpurun_out/r02gg
O=gpurun_out/r02gg
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
B="--steps 10 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws 8"
timeout 300 python bench.py $B > $O/b1.json 2>/dev/null
timeout 300 python bench.py $B > $O/b2.json 2>/dev/null
tail -2 $O/pytest.txt
python -c "
import json
for f in ['b1','b2']:
    d=json.loads(open('$O/'+f+'.json').read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['shard_projection']['per_w']['8']['projected_speedup'],3), round(d['shard_projection']['per_w']['8']['max_ms'],4))
"

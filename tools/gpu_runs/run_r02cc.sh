mkdir -p gpurun_out/r02cc
O=gpurun_out/r02cc
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/nvsmi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 666 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python -c "
import json
for f in ['bench_c4','bench_c5','bench_ref']:
    d=json.loads(open('$O/'+f+'.json').read().strip().splitlines()[-1]); print(f, d.get('value'), d.get('ms_per_step'), d.get('prep_ms'), (d.get('roofline') or {}).get('frac'), d.get('allocation_ms'), {w:round(v['projected_speedup'],3) for w,v in (d.get('shard_projection') or {}).get('per_w',{}).items()})
"

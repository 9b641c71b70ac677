mkdir -p gpurun_out/r02u
O=gpurun_out/r02u
timeout 300 python tools/shard_prof.py C4 1 8:7 > $O/shard.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws 8 > $O/bench_min.json 2> $O/bench_min.err
timeout 600 python bench.py --steps 10 --warmup 3 --shard-ws 8 > $O/bench_full.json 2> $O/bench_full.err
cat $O/shard.txt
python -c "
import json
for f in ['bench_min','bench_full']:
    d=json.loads(open('$O/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['prep_ms'], d['roofline']['kernel_ms'], d['shard_projection']['per_w']['8']['projected_speedup'])
"

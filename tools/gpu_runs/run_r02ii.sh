mkdir -p gpurun_out/r02ii
O=gpurun_out/r02ii
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python tools/shard_prof.py C4 1 8 > $O/shard.txt 2>&1
tail -2 $O/pytest.txt
python -c "
import json
d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['prep_ms'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['allocation_ms'], {w:round(v['projected_speedup'],3) for w,v in d['shard_projection']['per_w'].items()})
"
cat $O/shard.txt

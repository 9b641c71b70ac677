mkdir -p gpurun_out/r02kk
O=gpurun_out/r02kk
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
COSCHED_PAIR_TAIL_CONC=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fake or shard or tiled or c4 or C4" > $O/pytest_serial.txt 2>&1
timeout 300 python tools/shard_prof.py C4 1 8 > $O/shard.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
tail -2 $O/pytest.txt; tail -1 $O/pytest_serial.txt; cat $O/shard.txt | awk '{print $1,$2,$7,$8,$9}'
python -c "
import json
d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['prep_ms'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['allocation_ms'], {w:round(v['projected_speedup'],3) for w,v in d['shard_projection']['per_w'].items()})
"

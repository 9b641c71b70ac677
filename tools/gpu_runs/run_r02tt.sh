mkdir -p gpurun_out/r02tt
O=gpurun_out/r02tt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 666 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"score_triples_tiled" -c 1 -o $O/prof_c5 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > $O/ncu.log 2>&1
tail -2 $O/pytest.txt
python -c "
import json; d=json.loads(open('$O/bench_c5.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['allocation_ms'], {w:round(v['projected_speedup'],3) for w,v in d['shard_projection']['per_w'].items()})"

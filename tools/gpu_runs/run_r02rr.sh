mkdir -p gpurun_out/r02rr
O=gpurun_out/r02rr
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1
for v in pair plane; do
  if [ $v = plane ]; then E="COSCHED_TRIPLE_PLANE_ORDER=1"; else E="COSCHED_NOTHING=1"; fi
  env $E timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score_triples_tiled" -c 1 --csv --log-file $O/dram_c5_$v.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > /dev/null 2>&1
  env $E timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 > $O/bench_c5_$v.json 2>/dev/null
done
tail -2 $O/pytest.txt
for v in pair plane; do grep -h "dram__bytes\|gpu__time" $O/dram_c5_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'; python -c "
import json; d=json.loads(open('$O/bench_c5_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['shard_projection']['per_w']['8']['projected_speedup'])"; done

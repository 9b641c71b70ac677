mkdir -p gpurun_out/s1
for v in default plain; do
  if [ $v = default ]; then unset COSCHED_LIB_PATH; else export COSCHED_LIB_PATH=$PWD/tools/variants/$v.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws "" > gpurun_out/s1/c4_$v.json 2>/dev/null
  timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws "" > gpurun_out/s1/c5_$v.json 2>/dev/null
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tiled" -c 2 --csv --log-file gpurun_out/s1/c5_dram_$v.csv python bench.py --config C5 --steps 1 --warmup 1 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws "" > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tiled" -c 2 --csv --log-file gpurun_out/s1/c4_dram_$v.csv python bench.py --steps 1 --warmup 1 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws "" > /dev/null 2>&1
done
for f in gpurun_out/s1/*.json; do python -c "import json; d=json.loads(open('$f').read().strip().split('\n')[-1]); print('$f', d['value'], d['roofline']['kernel_ms'])"; done

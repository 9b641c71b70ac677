mkdir -p gpurun_out/v1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -q -x -k "not every_set" > gpurun_out/v1/tests.txt 2>&1
for v in default noflag; do
  if [ $v = default ]; then unset COSCHED_LIB_PATH; else export COSCHED_LIB_PATH=$PWD/tools/variants/$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/v1/launch_$v.csv python bench.py --steps 2 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 --shard-steps 1 > /dev/null 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 > gpurun_out/v1/bench_$v.json 2>/dev/null
done
unset COSCHED_LIB_PATH
tail -n 3 gpurun_out/v1/tests.txt

mkdir -p gpurun_out/v5
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_exactness.py -q -x -k "not every_set" > gpurun_out/v5/tests.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/v5/launch.csv python bench.py --steps 2 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 --shard-steps 1 > /dev/null 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 2,4,8 > gpurun_out/v5/bench.json 2>gpurun_out/v5/bench.err
tail -n 3 gpurun_out/v5/tests.txt

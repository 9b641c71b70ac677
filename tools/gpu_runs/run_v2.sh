mkdir -p gpurun_out/v2
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/v2/tests.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 24 --csv --log-file gpurun_out/v2/launch.csv python bench.py --steps 2 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 --shard-steps 1 > /dev/null 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 2,4,8 > gpurun_out/v2/bench.json 2>gpurun_out/v2/bench.err
timeout 300 ncu --set full --clock-control none -k regex:"merge_finish|k_gather|k_project" -c 3 -o gpurun_out/v2/prof_tail python bench.py --steps 1 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 --shard-steps 1 > gpurun_out/v2/ncu_full.log 2>&1
tail -n 3 gpurun_out/v2/tests.txt

mkdir -p gpurun_out/lb3
COSCHED_NCCL_LIB=$PWD/tests/loopback/libloopback_nccl.so timeout 450 python tests/loopback_ranks.py 2 > gpurun_out/lb3/w2.txt 2>&1; echo "rc=$?" >> gpurun_out/lb3/w2.txt
timeout 300 python tools/greedy_stats.py C4 5000 > gpurun_out/lb3/gstats.txt 2>&1
for sp in 1 0; do
  if [ $sp = 1 ]; then export COSCHED_PAIR_SPLIT=1; else unset COSCHED_PAIR_SPLIT; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/lb3/launch_split$sp.csv python bench.py --steps 2 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 --shard-steps 1 > /dev/null 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 --shard-ws 8 > gpurun_out/lb3/bench_split$sp.json 2>/dev/null
done
tail -n 5 gpurun_out/lb3/w2.txt gpurun_out/lb3/gstats.txt

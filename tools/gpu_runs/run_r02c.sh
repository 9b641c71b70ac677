mkdir -p gpurun_out/r02c
timeout 600 python tools/shard_prof.py C4 1 2 3 4 5 6 7 8 10 12 > gpurun_out/r02c/shard.txt 2>&1
COSCHED_PAIR_SPLIT=1 timeout 600 python tools/shard_prof.py C4 8 > gpurun_out/r02c/shard_nosplit.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c/c4_alloc_launches.csv python tools/alloc_prof.py C4 5000 > gpurun_out/r02c/alloc_ncu.log 2>&1
COSCHED_GREEDY_STATS=1 python tools/alloc_prof.py C4 5000 > gpurun_out/r02c/alloc_stats.txt 2>&1
tail -5 gpurun_out/r02c/shard.txt

mkdir -p gpurun_out/r02dd
O=gpurun_out/r02dd
COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C4 5000 1 > $O/c4_stats.txt 2>&1
COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C5 666 1 > $O/c5_stats.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_alloc.csv python tools/alloc_prof.py C4 5000 1 > /dev/null 2>&1
cat $O/c4_stats.txt $O/c5_stats.txt

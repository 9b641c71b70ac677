mkdir -p gpurun_out/r02j
O=gpurun_out/r02j
COSCHED_LIB_PATH=tools/variants/scanprof.so COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C4 5000 > $O/alloc.txt 2>&1
COSCHED_LIB_PATH=tools/variants/scanprof.so COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C5 666 >> $O/alloc.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/w8r7_launches.csv python tools/shard_prof.py C4 8:7 > $O/w8r7.txt 2>&1
timeout 300 python tools/shard_prof.py C4 8 > $O/w8.txt 2>&1
cat $O/alloc.txt; cat $O/w8.txt

mkdir -p gpurun_out/g6
export COSCHED_GREEDY_WIN0=65536 COSCHED_GREEDY_CHUNK=1048576
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g6/alloc_launches.csv python tools/alloc_prof.py C4 5000 > gpurun_out/g6/run.txt 2>&1
cat gpurun_out/g6/run.txt | tail -3

mkdir -p gpurun_out/g8
export COSCHED_GREEDY_WIN0=65536 COSCHED_GREEDY_CHUNK=1048576
timeout 600 ncu --set full --import-source on --clock-control none -k regex:greedy_scan -s 12 -c 1 -o gpurun_out/g8/scan python tools/alloc_prof.py C4 5000 > gpurun_out/g8/run.txt 2>&1
tail -2 gpurun_out/g8/run.txt

mkdir -p gpurun_out/g5
export COSCHED_GREEDY_STATS=1
for w0 in 4096 16384 65536; do for ch in 262144 1048576; do echo "win0 $w0 win $ch"; COSCHED_GREEDY_WIN0=$w0 COSCHED_GREEDY_CHUNK=$ch timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | tail -2; done; done > gpurun_out/g5/alloc.txt
cat gpurun_out/g5/alloc.txt

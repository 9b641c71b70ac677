mkdir -p gpurun_out/g7
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "greedy or c3 or alloc or c2 or fallback" > gpurun_out/g7/tests.txt 2>&1
export COSCHED_GREEDY_STATS=1
for w0 in 16384 65536; do for ch in 262144 1048576; do echo "win0 $w0 win $ch"; COSCHED_GREEDY_WIN0=$w0 COSCHED_GREEDY_CHUNK=$ch timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | tail -2; done; done > gpurun_out/g7/alloc.txt
timeout 120 python tools/alloc_prof.py C5 666 >> gpurun_out/g7/alloc.txt 2>&1
tail -n 2 gpurun_out/g7/tests.txt; cat gpurun_out/g7/alloc.txt

mkdir -p gpurun_out/g2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "greedy or c3 or alloc or c2" > gpurun_out/g2/tests.txt 2>&1
for ch in 65536 262144 1048576 4194304; do COSCHED_GREEDY_CHUNK=$ch timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | tail -1 | sed "s/^/chunk $ch: /"; done > gpurun_out/g2/alloc.txt
timeout 120 python tools/alloc_prof.py C5 666 >> gpurun_out/g2/alloc.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g2/alloc_launches.csv python tools/alloc_prof.py C4 5000 > /dev/null 2>&1
tail -n 3 gpurun_out/g2/tests.txt; cat gpurun_out/g2/alloc.txt

mkdir -p gpurun_out/g11
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or c3 or alloc or c2 or fallback or loopback" > gpurun_out/g11/tests.txt 2>&1
for p in 1 0; do echo "pipe $p"; COSCHED_GREEDY_PIPE=$p timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | tail -1; COSCHED_GREEDY_PIPE=$p timeout 300 python tools/alloc_prof.py C5 666 2>&1 | tail -1; done > gpurun_out/g11/alloc.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g11/alloc_launches.csv python tools/alloc_prof.py C4 5000 > /dev/null 2>&1
tail -n 3 gpurun_out/g11/tests.txt; cat gpurun_out/g11/alloc.txt

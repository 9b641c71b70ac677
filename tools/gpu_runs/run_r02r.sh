mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or alloc or fallback or loopback" > $O/tests.txt 2>&1
COSCHED_GREEDY_STATS=1 COSCHED_LIB_PATH=tools/variants/scanprof.so timeout 300 python tools/alloc_prof.py C4 5000 > $O/alloc.txt 2>&1
timeout 300 python tools/alloc_prof.py C4 5000 >> $O/alloc.txt 2>&1
timeout 300 python tools/alloc_prof.py C5 666 >> $O/alloc.txt 2>&1
tail -2 $O/tests.txt; cat $O/alloc.txt

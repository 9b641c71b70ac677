mkdir -p gpurun_out/r02m
O=gpurun_out/r02m
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py tests/test_gpu_loopback.py -q -x > $O/tests.txt 2>&1
timeout 300 python tools/shard_prof.py C4 1 4 8 10 > $O/conc.txt 2>&1
COSCHED_PAIR_TAIL_CONC=0 timeout 300 python tools/shard_prof.py C4 1 4 8 10 > $O/noconc.txt 2>&1
tail -n 2 $O/tests.txt; paste -d'\n' $O/conc.txt $O/noconc.txt

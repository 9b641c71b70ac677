mkdir -p gpurun_out/r02ll
O=gpurun_out/r02ll
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or alloc or fallback or loopback" > $O/tests.txt 2>&1
COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C4 5000 1 > $O/c4_stats.txt 2>&1
timeout 300 python tools/alloc_prof.py C4 5000 8 | tail -1 > $O/alloc.txt 2>&1
timeout 300 python tools/alloc_prof.py C5 666 4 | tail -1 >> $O/alloc.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"obj_hist" --csv --log-file $O/hist.csv python tools/alloc_prof.py C5 666 1 > /dev/null 2>&1
tail -2 $O/tests.txt; cat $O/c4_stats.txt $O/alloc.txt; grep obj_hist $O/hist.csv | head -4

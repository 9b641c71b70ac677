mkdir -p gpurun_out/r02mm
O=gpurun_out/r02mm
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or alloc or fallback or loopback or triple" > $O/tests.txt 2>&1
timeout 300 python tools/alloc_prof.py C5 666 4 | tail -1 > $O/alloc.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"keys_live" --csv --log-file $O/live.csv python tools/alloc_prof.py C5 666 1 > /dev/null 2>&1
tail -2 $O/tests.txt; cat $O/alloc.txt; grep "gpu__time" $O/live.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,100-

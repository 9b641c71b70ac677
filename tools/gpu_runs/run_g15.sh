mkdir -p gpurun_out/g15
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "greedy or c3 or alloc or fallback" > gpurun_out/g15/tests.txt 2>&1
timeout 300 python tools/alloc_prof.py C5 666 > gpurun_out/g15/alloc.txt 2>&1
timeout 120 python tools/alloc_prof.py C4 5000 >> gpurun_out/g15/alloc.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"keys_in_range|keys_live" --csv --log-file gpurun_out/g15/kir.csv python tools/alloc_prof.py C5 666 > /dev/null 2>&1
tail -n 2 gpurun_out/g15/tests.txt; cat gpurun_out/g15/alloc.txt

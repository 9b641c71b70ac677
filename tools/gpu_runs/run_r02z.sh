mkdir -p gpurun_out/r02z
O=gpurun_out/r02z
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"keys_in_range|keys_live|obj_hist|obj_minmax|select_free|k_greedy_scan" --csv --log-file $O/c5_kir.csv python tools/alloc_prof.py C5 666 1 > $O/c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"keys_in_range|keys_live|obj_hist|obj_minmax" --csv --log-file $O/c4_kir.csv python tools/alloc_prof.py C4 5000 1 > $O/c4.log 2>&1
ls -la $O

mkdir -p gpurun_out/r02aa
O=gpurun_out/r02aa
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or alloc or fallback or loopback" > $O/tests.txt 2>&1
for ch in 262144 1048576 4194304; do
  echo "== window max $ch" >> $O/alloc.txt
  COSCHED_GREEDY_CHUNK=$ch timeout 300 python tools/alloc_prof.py C4 5000 6 | tail -1 >> $O/alloc.txt 2>&1
  COSCHED_GREEDY_CHUNK=$ch timeout 300 python tools/alloc_prof.py C5 666 4 | tail -1 >> $O/alloc.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"keys_live" --csv --log-file $O/live.csv python tools/alloc_prof.py C5 666 1 > /dev/null 2>&1
tail -2 $O/tests.txt; cat $O/alloc.txt

mkdir -p gpurun_out/r02q
O=gpurun_out/r02q
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or alloc or fallback or loopback" > $O/tests.txt 2>&1
for v in tiled cub; do
  if [ $v = cub ]; then E="COSCHED_GREEDY_CUBSELECT=1"; else E="COSCHED_NOTHING=1"; fi
  echo "== $v" >> $O/alloc.txt
  env $E timeout 300 python tools/alloc_prof.py C4 5000 >> $O/alloc.txt 2>&1
  env $E timeout 300 python tools/alloc_prof.py C5 666 >> $O/alloc.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_alloc_launches.csv python tools/alloc_prof.py C4 5000 > /dev/null 2>&1
tail -2 $O/tests.txt; cat $O/alloc.txt

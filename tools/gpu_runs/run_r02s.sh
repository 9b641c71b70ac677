mkdir -p gpurun_out/r02s
O=gpurun_out/r02s
for v in lookback cub; do
  if [ $v = cub ]; then E="COSCHED_GREEDY_CUBSELECT=1"; else E="COSCHED_NOTHING=1"; fi
  echo "== $v" >> $O/alloc.txt
  env $E timeout 300 python tools/alloc_prof.py C4 5000 8 | tail -1 >> $O/alloc.txt 2>&1
  env $E timeout 300 python tools/alloc_prof.py C5 666 6 | tail -1 >> $O/alloc.txt 2>&1
done
cat $O/alloc.txt

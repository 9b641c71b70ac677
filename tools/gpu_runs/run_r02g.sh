mkdir -p gpurun_out/r02g
O=gpurun_out/r02g
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "greedy or alloc or fallback or loopback" > $O/tests.txt 2>&1
for v in default scanprof scanold; do
  if [ $v = default ]; then L=""; else L="COSCHED_LIB_PATH=tools/variants/$v.so"; fi
  echo "== $v" >> $O/alloc.txt
  env $L COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C4 5000 >> $O/alloc.txt 2>&1
  env $L COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C5 666 >> $O/alloc.txt 2>&1
done
tail -3 $O/tests.txt; cat $O/alloc.txt

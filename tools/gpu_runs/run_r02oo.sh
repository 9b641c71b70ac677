mkdir -p gpurun_out/r02oo
O=gpurun_out/r02oo
for w0 in 8192 16384 65536; do
  for ch in 131072 262144 524288; do
    echo "win0=$w0 max=$ch $(COSCHED_GREEDY_WIN0=$w0 COSCHED_GREEDY_CHUNK=$ch timeout 300 python tools/alloc_prof.py C4 5000 6 | tail -1)" >> $O/sweep.txt
  done
done
cat $O/sweep.txt

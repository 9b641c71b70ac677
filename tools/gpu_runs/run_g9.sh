mkdir -p gpurun_out/g9
export COSCHED_GREEDY_STATS=1
for v in scan4 scan8 default; do
  if [ $v = default ]; then unset COSCHED_LIB_PATH; else export COSCHED_LIB_PATH=$PWD/tools/variants/$v.so; fi
  for w0 in 16384 65536; do for ch in 262144 1048576; do echo "$v win0 $w0 win $ch"; COSCHED_GREEDY_WIN0=$w0 COSCHED_GREEDY_CHUNK=$ch timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | tail -1; done; done
done > gpurun_out/g9/alloc.txt
cat gpurun_out/g9/alloc.txt

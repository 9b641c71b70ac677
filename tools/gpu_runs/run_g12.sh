mkdir -p gpurun_out/g12
export COSCHED_GREEDY_STATS=1
for v in ahead2 ahead4 ahead8 ahead16; do export COSCHED_LIB_PATH=$PWD/tools/variants/$v.so; echo "== $v"; timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | tail -7; done > gpurun_out/g12/alloc.txt
cat gpurun_out/g12/alloc.txt

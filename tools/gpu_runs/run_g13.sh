mkdir -p gpurun_out/g13
export COSCHED_GREEDY_STATS=1
for v in p2a2 p2a4 p4a2 p4a1; do export COSCHED_LIB_PATH=$PWD/tools/variants/$v.so; echo "== $v"; timeout 120 python tools/alloc_prof.py C4 5000 2>&1 | grep -E "allocation|survivors" | tail -6; done > gpurun_out/g13/alloc.txt
cat gpurun_out/g13/alloc.txt

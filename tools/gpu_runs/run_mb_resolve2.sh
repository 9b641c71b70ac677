mkdir -p gpurun_out/mb
./tools/microbench/resolve2 > gpurun_out/mb/resolve2.txt 2>&1
cat gpurun_out/mb/resolve2.txt

mkdir -p gpurun_out/mb
./tools/microbench/resolve > gpurun_out/mb/resolve.txt 2>&1
cat gpurun_out/mb/resolve.txt

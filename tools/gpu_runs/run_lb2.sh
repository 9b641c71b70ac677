mkdir -p gpurun_out/lb2
python -c "import sys; sys.path.insert(0,'tests'); import loopback; print(loopback.build())" > gpurun_out/lb2/build.txt 2>&1
COSCHED_NCCL_LIB=$PWD/tests/loopback/libloopback_nccl.so timeout 450 python tests/loopback_ranks.py 2 > gpurun_out/lb2/w2.txt 2>&1; echo "rc=$?" >> gpurun_out/lb2/w2.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "split or fake or hand or c3" > gpurun_out/lb2/split.txt 2>&1
timeout 300 python tools/greedy_stats.py C4 5000 > gpurun_out/lb2/gstats.txt 2>&1
timeout 300 python bench.py --no-hill --calib-coruns 0 --no-cpu-baseline > gpurun_out/lb2/bench.json 2> gpurun_out/lb2/bench.err
tail -n 5 gpurun_out/lb2/w2.txt gpurun_out/lb2/split.txt gpurun_out/lb2/gstats.txt

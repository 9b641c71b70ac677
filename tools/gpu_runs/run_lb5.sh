mkdir -p gpurun_out/lb5
export COSCHED_NCCL_LIB=$PWD/tests/loopback/libloopback_nccl.so
python -c "import sys; sys.path.insert(0,'tests'); import loopback; loopback.build()"
timeout 300 python tests/loopback_ranks.py 2 > gpurun_out/lb5/w2.txt 2>&1; echo "rc=$?" >> gpurun_out/lb5/w2.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tests/loopback_ranks.py 2 > gpurun_out/lb5/memcheck.txt 2>&1
tail -n 30 gpurun_out/lb5/w2.txt; grep -m 20 -E "Invalid|at 0x|by thread|in k_|cosched::" gpurun_out/lb5/memcheck.txt | head -30

mkdir -p gpurun_out/r02a
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02a/pytest.txt 2>&1
bash tools/gpu_bench_profile.sh r02a_prof > gpurun_out/r02a/prof.log 2>&1
tail -n 3 gpurun_out/r02a/pytest.txt

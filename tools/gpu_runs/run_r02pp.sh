mkdir -p gpurun_out/r02pp
timeout 600 python -m pytest tests/test_gpu_api.py -q > gpurun_out/r02pp/t.txt 2>&1
tail -15 gpurun_out/r02pp/t.txt

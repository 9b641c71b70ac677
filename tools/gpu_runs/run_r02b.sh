mkdir -p gpurun_out/r02b
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02b/pytest.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err
timeout 300 python tools/alloc_prof.py C4 5000 > gpurun_out/r02b/alloc.txt 2>&1
tail -n 3 gpurun_out/r02b/pytest.txt; tail -c 600 gpurun_out/r02b/bench.json; cat gpurun_out/r02b/alloc.txt | tail -20

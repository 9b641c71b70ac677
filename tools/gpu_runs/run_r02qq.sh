mkdir -p gpurun_out/r02qq
O=gpurun_out/r02qq
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.txt 2>&1
timeout 1500 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > $O/bench_c5.json 2> $O/bench_c5.err
tail -2 $O/pytest.txt; tail -c 300 $O/bench_c5.json

mkdir -p gpurun_out/r02l
O=gpurun_out/r02l
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 > $O/bench.json 2> $O/bench.err
timeout 300 python tools/shard_prof.py C4 8 > $O/w8.txt 2>&1
tail -n 3 $O/pytest.txt; cat $O/w8.txt

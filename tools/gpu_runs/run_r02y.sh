mkdir -p gpurun_out/r02y
O=gpurun_out/r02y
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 300 python tools/shard_prof.py C4 1 8 > $O/shard.txt 2>&1
COSCHED_PREP_EVENTS=1 timeout 300 python tools/shard_prof.py C4 8:0 8:7 2> $O/prep.txt > /dev/null
tail -n 2 $O/pytest.txt; cat $O/shard.txt; tail -4 $O/prep.txt

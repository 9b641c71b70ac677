mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 300 python tools/shard_prof.py C4 1 8 > $O/split.txt 2>&1
COSCHED_SPLIT_GATHER=0 timeout 300 python tools/shard_prof.py C4 1 8 > $O/nosplit.txt 2>&1
timeout 300 python tools/shard_prof.py C4 1 8 > $O/split2.txt 2>&1
tail -n 2 $O/pytest.txt; cat $O/split.txt $O/nosplit.txt $O/split2.txt

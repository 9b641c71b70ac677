mkdir -p gpurun_out/r02jj
O=gpurun_out/r02jj
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
COSCHED_PAIR_ONE_LAUNCH=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_old.txt 2>&1
timeout 300 python tools/shard_prof.py C4 1 8 > $O/shard.txt 2>&1
COSCHED_PAIR_ONE_LAUNCH=0 timeout 300 python tools/shard_prof.py C4 1 8 > $O/shard_old.txt 2>&1
tail -2 $O/pytest.txt; tail -1 $O/pytest_old.txt; paste -d'|' $O/shard.txt $O/shard_old.txt | awk -F'|' '{split($1,a," "); split($2,b," "); print a[1],a[2],a[7],b[7]}'

mkdir -p gpurun_out/r02v
O=gpurun_out/r02v
COSCHED_PREP_EVENTS=1 timeout 300 python tools/shard_prof.py C4 1 8:0 8:7 > $O/shard.txt 2> $O/prep.txt
cat $O/shard.txt; tail -8 $O/prep.txt

#!/bin/bash
# C5 (triples): bench line + ncu launch list + full capture of the triple scorer.
OUT=gpurun_out/${1:-c5}
mkdir -p $OUT
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --alloc-k 666 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $OUT/launches.csv \
    python bench.py --config C5 --steps 1 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score -s 3 -c 1 -o $OUT/prof_score \
    python bench.py --config C5 --steps 1 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 > $OUT/ncu_full_run.log 2>&1
ls -la $OUT

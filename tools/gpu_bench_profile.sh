#!/bin/bash
# One GPU round: tests, bench, ncu launch list + full capture of the scorer.
# usage: bash tools/gpu_bench_profile.sh <tag> [extra bench args]
set -x
TAG=${1:-run}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/nvsmi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 "$@" > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 "$@" > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pairs_tiled<\(int\)2, \(int\)4, \(bool\)0>|triples_tiled" -s 2 -c 1 -o $OUT/prof_score \
    python bench.py --steps 1 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 "$@" > $OUT/ncu_full_run.log 2>&1
ls -la $OUT

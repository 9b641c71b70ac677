#!/bin/bash
# ncu --set full of the projection/gather kernels (C4), one launch each.
OUT=gpurun_out/${1:-prep}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_project_all|k_gather_fast" -s 6 -c 2 -o $OUT/prof_prep \
    python bench.py --steps 1 --warmup 3 --alloc-k 0 --no-cpu-baseline --no-hill --calib-coruns 0 > $OUT/ncu_prep_run.log 2>&1
ls -la $OUT

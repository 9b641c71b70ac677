#!/bin/bash
# run on the GPU box: plain timing, then ncu per-pipe counters
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
./pipes | tee ../../gpurun_out/pipes_plain.txt
ncu --clock-control none --metrics sm__inst_executed.avg.per_cycle_active,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --csv ./pipes > ../../gpurun_out/pipes_ncu.csv 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> ../../gpurun_out/pipes_plain.txt

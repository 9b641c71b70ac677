#!/bin/bash
# run on the GPU box: timing, then shared-memory wavefronts per load instruction
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
./lds | tee ../../gpurun_out/lds_plain.txt
ncu --clock-control none --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum --csv ./lds > ../../gpurun_out/lds_ncu.csv 2>&1

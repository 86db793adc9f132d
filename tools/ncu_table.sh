#!/bin/bash
# Per-kernel ncu metrics of tools/profile_workload.py (under gpurun, 1 GPU).
TAG=${1:-r2}
KIND=${2:-cfg2}
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
mkdir -p gpurun_out
timeout 1200 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ncu_table_$TAG.csv python tools/profile_workload.py $KIND --range \
  > gpurun_out/ncu_table_$TAG.log 2>&1
echo "ncu-table rc=$?"

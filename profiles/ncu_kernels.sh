#!/bin/bash
# Per-kernel instruction / time / traffic of a short c2 query batch (direct launches, serialised by ncu).
set -e
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_pipe_lsu.sum,smsp__inst_executed_pipe_fp64.sum
PROBE_NQ=${PROBE_NQ:-100} ncu --profile-from-start off --clock-control none --metrics "$M" --csv \
  --log-file gpurun_out/ncu_kernels.csv python profiles/graph_probe.py > gpurun_out/ncu_kernels.log 2>&1

#!/bin/bash
# Whole-batch metrics of one concurrent c2 query batch (graph workload).
# Run on the GPU box from the repo root, after profiles/graph_probe.py ran clean.
set -e
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
M=$M,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,dram__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_elapsed
M=$M,smsp__inst_executed.sum,smsp__inst_executed_pipe_lsu.sum
M=$M,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
M=$M,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for s in long_scoreboard short_scoreboard mio_throttle lg_throttle barrier membar no_instruction math_pipe_throttle \
         not_selected selected wait branch_resolving dispatch_stall drain misc; do
  M=$M,smsp__average_warps_issue_stalled_${s}_per_issue_active.ratio
done
TSG_GRAPHS=1 ncu --profile-from-start off --graph-profiling graph \
  --clock-control none --metrics "$M" --csv --log-file gpurun_out/ncu_graph.csv \
  python profiles/graph_probe.py > gpurun_out/ncu_graph.log 2>&1

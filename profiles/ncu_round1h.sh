#!/bin/bash
# Round-1h ncu evidence (final round-1 code: u16x2 box clamps, CUDA-graph pipeline, one reservation per stage flush); run under gpurun from the repo root, one GPU.
#  1. plain run of the bench command (must exit 0 first),
#  2. launch list: every kernel launch with its device time and DRAM bytes (cold-cache,
#     serialised: compare SHARES, not absolutes),
#  3. one --set full capture per hot kernel of the first timed step (K1: the timed build, not the
#     1M-series warm-up build)
#     (warm-up = 3 steps; lbscan / refine launch twice per step).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_summarise -s 1 -c 1 \
    -o gpurun_out/prof_k_summarise -f $CMD > gpurun_out/ncu_k1.log 2>&1
for k in k_groups k_bound; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o gpurun_out/prof_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
done
for k in k_lbscan k_refine_tma; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 2 \
      -o gpurun_out/prof_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
done

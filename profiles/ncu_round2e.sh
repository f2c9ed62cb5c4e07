#!/bin/bash
# Round-2e ncu evidence (final round-2 code: block-wide query selection, surplus blocks retired, weighted refinement start,
# bound / lbscan at 4 blocks per SM with register-held shared addresses, 4 group boxes per thread); run under gpurun, one GPU.
#  1. plain run of the bench command (must exit 0 first),
#  2. launch list: every kernel launch with its device time and DRAM bytes (cold-cache,
#     serialised: compare SHARES, not absolutes),
#  3. one --set full capture per hot kernel of the first timed batch (parity batch + 3 warm-up
#     batches come first; bound / lbscan / refine launch twice per batch), K1 and the K2 gather of
#     the timed build (the 1M-series warm-up build comes first).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs"
$CMD > gpurun_out/ncu_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r2e.csv $CMD > gpurun_out/ncu_launches.log 2>&1
for k in k_summarise k_gather_words; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/r2e_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_groups -s 4 -c 1 \
    -o gpurun_out/r2e_k_groups -f $CMD > gpurun_out/ncu_k_groups.log 2>&1
for k in k_bound k_lbscan k_refine_tma; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 2 \
      -o gpurun_out/r2e_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
done

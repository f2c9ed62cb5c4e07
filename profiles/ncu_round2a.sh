#!/bin/bash
# Round-2a ncu evidence: --set full with source of the first timed batch's lbscan / refine / bound
# launches (parity batch + 3 warm-up batches = 8 launches of each before it; wave 1 = the 10th).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1
for k in k_lbscan k_refine_tma k_bound; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 2 \
      -o gpurun_out/r2a_$k -f $CMD > gpurun_out/ncu_r2a_$k.log 2>&1
done

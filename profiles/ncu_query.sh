#!/bin/bash
# ncu captures of the query kernels at c2 scale (100M x 256), one GPU.
set -e
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1
for k in k_bound k_seed k_lbscan k_refine; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 2 -o gpurun_out/prof_$k $CMD > gpurun_out/ncu_$k.log 2>&1
done

#!/bin/bash
# ncu --set full of both lbscan launches of the first timed step at c4 (1 GPU share: 125M x 96 mixture).
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/c4_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_lbscan -s 6 -c 2 \
    -o gpurun_out/prof_lbscan_c4 -f $CMD > gpurun_out/ncu_lbscan_c4.log 2>&1

#!/bin/bash
# ncu --set full of the wave-B refinement launch of the first timed step at c5 sigma=0.5, batch 64
# (hard queries: refinement dominates). Run under gpurun from the repo root, one GPU.
mkdir -p gpurun_out
CMD="python bench.py --config c5 --sigma 0.5 --batch 64 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/c5_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_refine_tma -s 7 -c 1 \
    -o gpurun_out/prof_refine_c5 -f $CMD > gpurun_out/ncu_refine_c5.log 2>&1

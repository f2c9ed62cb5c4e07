#!/bin/bash
# ncu captures for round 1 (run under gpurun from the repo root).
# Plain run first (must exit 0), then one full-set capture per hot kernel.
set -e
CMD="python bench.py --count 20000000 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_summarise -c 1 -o gpurun_out/prof_k1 $CMD > gpurun_out/ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lbscan -s 200 -c 2 -o gpurun_out/prof_lbscan $CMD > gpurun_out/ncu_lbscan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_refine -s 400 -c 2 -o gpurun_out/prof_refine $CMD > gpurun_out/ncu_refine.log 2>&1

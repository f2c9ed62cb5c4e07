#!/bin/bash
# A/B (round 2, final kernels): bound's pages per lane (TSG_BOUND_PL) and blocks per SM.
mkdir -p gpurun_out
for r in 1 2; do
  python bench.py --no-cpu-baseline --no-other-configs --steps 20 --warmup 5 > gpurun_out/ab_t3_default_$r.log 2>&1
  for v in bpl1 bpl4 mb6 mb4; do
    TSG_LIB_PATH=paper_2009_00786_b200/_variants/$v.so python bench.py --no-cpu-baseline --no-other-configs \
      --steps 20 --warmup 5 > gpurun_out/ab_t3_${v}_$r.log 2>&1
  done
done

#!/bin/bash
# A/B (round 2): sorted key width (TSG_SORT_BITS) 48 (default) vs 56 vs 64: build time vs query rate.
mkdir -p gpurun_out
for b in 48 56 64; do
  TSG_SORT_BITS=$b python bench.py --no-cpu-baseline --no-other-configs --steps 20 --warmup 5 > gpurun_out/ab_sb_$b.log 2>&1
done

#!/bin/bash
# A/B (round 2): wave split fraction (TSG_REFINE_SPLIT) with the split refinement kernels of that build
# (since removed), and the fused kernel (TSG_REFINE_FUSED, then an env switch). Result: split 0.3 best
# (0.15: 27.7K q/s, 0.2: 31.7K, 0.3: 33.4K, 0.45: 30.9K); the fused kernel 33.8K.
mkdir -p gpurun_out
for sp in 0.15 0.2 0.3 0.45; do
  TSG_REFINE_SPLIT=$sp python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_split_$sp.log 2>&1
done
TSG_REFINE_FUSED=1 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_split_fused.log 2>&1

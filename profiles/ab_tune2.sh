#!/bin/bash
# A/B (round 2, after the index-order fine summary): occupancy / chunk knobs of bound, lbscan, refine.
mkdir -p gpurun_out
for r in 1 2; do
  python bench.py --no-cpu-baseline --no-other-configs --steps 20 --warmup 5 > gpurun_out/ab_t2_default_$r.log 2>&1
  for v in fc256 mb3 mb5 ml4 ml6; do
    TSG_LIB_PATH=paper_2009_00786_b200/_variants/$v.so python bench.py --no-cpu-baseline --no-other-configs \
      --steps 20 --warmup 5 > gpurun_out/ab_t2_${v}_$r.log 2>&1
  done
done

#!/bin/bash
# A/B (round 2): fused refinement at 3 blocks/SM with a half-precision fine table (default) vs
# round 1's configuration (float table, 2 blocks/SM, 128-record chunks), 128-record chunks at 3/SM,
# and the split kernels (a fine-filter kernel writing survivor lists, then a row kernel over them;
# TSG_REFINE_SPLIT_KERNELS=1 in the build of that run, since removed).
# Result (same box): r1 34.07K q/s (wave B 4.50 us/query), 3/SM + chunk 128 33.9K (4.58),
# 3/SM + chunk 64 33.1K (5.46), split 33.6K (4.58, wave A 1.30 vs 1.02). Round 1's config stays.
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3.log
for r in 1 2; do
  python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_r3_default_$r.log 2>&1
  TSG_LIB_PATH=paper_2009_00786_b200/_variants/r1refine.so python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_r3_r1_$r.log 2>&1
  TSG_LIB_PATH=paper_2009_00786_b200/_variants/m3c128.so python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_r3_c128_$r.log 2>&1
  TSG_REFINE_SPLIT_KERNELS=1 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_r3_split_$r.log 2>&1
done

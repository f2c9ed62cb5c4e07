#!/bin/bash
# A/B: w = 16 box bounds with native u16x2 clamps (default build) vs byte-SIMD
# __vmaxu4 / __vminu4 (variant old_box: bash profiles/build_variant.sh old_box -DTSG_BOX_U16=0).
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_u16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_u16.log
for r in 1 2; do
  python bench.py --no-cpu-baseline > gpurun_out/ab_u16_c2_$r.log 2>&1
  TSG_LIB_PATH=paper_2009_00786_b200/_variants/old_box.so python bench.py --no-cpu-baseline > gpurun_out/ab_old_c2_$r.log 2>&1
done
python bench.py --config c5 --sigma 0.5 --batch 64 --no-cpu-baseline > gpurun_out/ab_u16_c5.log 2>&1
TSG_LIB_PATH=paper_2009_00786_b200/_variants/old_box.so python bench.py --config c5 --sigma 0.5 --batch 64 --no-cpu-baseline > gpurun_out/ab_old_c5.log 2>&1

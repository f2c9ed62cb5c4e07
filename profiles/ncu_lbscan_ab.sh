#!/bin/bash
# ncu --set full of lbscan (both waves of the first timed batch) for the in-tree library and for
# variant builds. usage: bash profiles/ncu_lbscan_ab.sh [KERNEL_REGEX] NAME...  (default + variants)
k=${1:-k_lbscan}; shift
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs"
ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 2 \
    -o gpurun_out/ab_${k}_default -f $CMD > gpurun_out/ncu_ab_${k}_default.log 2>&1
for v in "$@"; do
  TSG_LIB_PATH=paper_2009_00786_b200/_variants/$v.so ncu --set full --clock-control none --import-source on \
    -k regex:$k -s 8 -c 2 -o gpurun_out/ab_${k}_$v -f $CMD > gpurun_out/ncu_ab_${k}_$v.log 2>&1
done
ls -la gpurun_out/*.ncu-rep

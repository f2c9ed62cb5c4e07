#!/bin/bash
# A/B (round 2): the L2 fetch granularity hint (cudaLimitMaxL2FetchGranularity, TSG_L2_FETCH) vs
# lbscan's DRAM bytes and the c2 query rate.
mkdir -p gpurun_out
TSG_PRINT_L2_FETCH=1 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_l2_default.log 2>&1
for g in 32 64 128; do
  TSG_L2_FETCH=$g python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_l2_$g.log 2>&1
done
for g in default 32 64; do
  if [ $g = default ]; then E=""; else E="TSG_L2_FETCH=$g"; fi
  env $E ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_lbscan -s 8 -c 2 --csv --log-file gpurun_out/ab_l2_ncu_$g.csv \
    python bench.py --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
done

#!/bin/bash
# A/B (round 2): lbscan's L2 prefetches. default = prefetch.global.L2 of the line; pf0 = none;
# pf2 = cp.async.bulk.prefetch.L2 of exactly the quad's words / the run's quad boxes.
# Variants: bash profiles/build_variant.sh pf0 -DTSG_PREFETCH=0; ... pf2 -DTSG_PREFETCH=2
mkdir -p gpurun_out
for r in 1 2; do
  for v in default pf0 pf2; do
    if [ $v = default ]; then L=""; else L=paper_2009_00786_b200/_variants/$v.so; fi
    TSG_LIB_PATH=$L python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_pf_${v}_$r.log 2>&1
  done
done
for v in default pf0 pf2; do
  if [ $v = default ]; then L=""; else L=paper_2009_00786_b200/_variants/$v.so; fi
  TSG_LIB_PATH=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    --clock-control none -k regex:k_lbscan -s 8 -c 4 --csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 \
    > gpurun_out/ab_pf_ncu_$v.csv 2> gpurun_out/ab_pf_ncu_$v.err
done

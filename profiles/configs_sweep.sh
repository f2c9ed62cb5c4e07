#!/bin/bash
# Every BASELINE config on one GPU (the c2 headline is bench.py's default run).
mkdir -p gpurun_out
for c in c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/sweep_$c.log 2>&1; done
for s in 0.01 0.1 0.5 1.0; do for b in 1 64 1024; do
  st=5; [ $b = 1 ] && st=50; [ $b = 1024 ] && st=2
  python bench.py --config c5 --sigma $s --batch $b --steps $st --no-cpu-baseline > gpurun_out/sweep_c5_${s}_$b.log 2>&1
done; done
python bench.py --config c1 --dtw 12 --no-cpu-baseline > gpurun_out/sweep_c1_dtw12.log 2>&1

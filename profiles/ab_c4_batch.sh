#!/bin/bash
# c4: slot size vs batch size (TSG_BATCH = slots per batch; fewer slots -> larger candidate
# capacity per slot -> fewer full-size reruns of overflowing queries).
mkdir -p gpurun_out
for b in 128 64 32; do
  TSG_BATCH=$b python bench.py --config c4 --no-cpu-baseline > gpurun_out/ab_c4_batch$b.log 2>&1
done

#!/bin/bash
# Batched rerun of overflowing queries: GPU tests, c4 / c5 sigma=1 / c2 benches (and c4 with the old one-query reruns).
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_rr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rr.log
python bench.py --config c4 --no-cpu-baseline > gpurun_out/rr_c4.log 2>&1
TSG_NO_BATCHED_RERUN=1 python bench.py --config c4 --no-cpu-baseline > gpurun_out/rr_c4_old.log 2>&1
python bench.py --config c5 --sigma 1.0 --batch 64 --no-cpu-baseline > gpurun_out/rr_c5s1_64.log 2>&1
python bench.py --config c5 --sigma 1.0 --batch 1024 --steps 2 --no-cpu-baseline > gpurun_out/rr_c5s1_1024.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/rr_c2.log 2>&1

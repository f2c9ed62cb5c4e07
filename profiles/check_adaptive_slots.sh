#!/bin/bash
# Overflow feedback (fewer, larger slots after a call with >5% overflowing queries): GPU tests,
# c4 (with and without the feedback), c5 sigma=1 batch 64, and the default c2 bench.
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_as.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_as.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_as.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_as.log
python bench.py --config c4 --no-cpu-baseline > gpurun_out/as_c4.log 2>&1
TSG_FIXED_BATCH=1 python bench.py --config c4 --no-cpu-baseline > gpurun_out/as_c4_fixed.log 2>&1
python bench.py --config c5 --sigma 1.0 --batch 64 --no-cpu-baseline > gpurun_out/as_c5s1_64.log 2>&1
python bench.py --config c5 --sigma 0.5 --batch 64 --no-cpu-baseline > gpurun_out/as_c5s05_64.log 2>&1
python bench.py > gpurun_out/as_c2.log 2>&1

#!/bin/bash
# One candidate-record reservation per lbscan stage flush: GPU tests, smoke, c4, c2, c5 sigma=1.
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_sr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sr.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_sr.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_sr.log
python bench.py --config c4 --no-cpu-baseline > gpurun_out/sr_c4.log 2>&1
python bench.py --config c5 --sigma 1.0 --batch 64 --no-cpu-baseline > gpurun_out/sr_c5s1_64.log 2>&1
python bench.py > gpurun_out/sr_c2.log 2>&1

#!/bin/bash
# A/B: the batch pipeline as a cached CUDA graph (default) vs plain stream launches (TSG_NO_GRAPH=1);
# c2 (batch 100) and c5 sigma=0.01 / 0.1 at batch 1 and 64 (launch-bound shapes).
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_graph.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_graph.log
python bench.py --no-cpu-baseline > gpurun_out/ab_graph_c2.log 2>&1
TSG_NO_GRAPH=1 python bench.py --no-cpu-baseline > gpurun_out/ab_nograph_c2.log 2>&1
for b in 1 64; do
  python bench.py --config c5 --sigma 0.01 --batch $b --no-cpu-baseline > gpurun_out/ab_graph_c5_b$b.log 2>&1
  TSG_NO_GRAPH=1 python bench.py --config c5 --sigma 0.01 --batch $b --no-cpu-baseline > gpurun_out/ab_nograph_c5_b$b.log 2>&1
done
python bench.py --config c5 --sigma 0.1 --batch 1 --no-cpu-baseline > gpurun_out/ab_graph_c5s01_b1.log 2>&1
TSG_NO_GRAPH=1 python bench.py --config c5 --sigma 0.1 --batch 1 --no-cpu-baseline > gpurun_out/ab_nograph_c5s01_b1.log 2>&1

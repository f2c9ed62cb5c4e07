#!/bin/bash
# One gpurun pass: GPU parity tests, then bench.py (default: c2) with any extra bench args.
# usage: bash profiles/gpu_check.sh TAG [extra bench args...]   (outputs in gpurun_out/*_TAG.*)
tag=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi_$tag.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_$tag.log
timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$tag.log

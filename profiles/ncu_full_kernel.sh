#!/bin/bash
# Full ncu section set for one launch of one kernel (regex $1, skip $2 launches) of the c2 probe batch.
set -e
mkdir -p gpurun_out
K=${1:-k_bound}; SKIP=${2:-3}; OUT=${3:-gpurun_out/full_$K}
PROBE_NQ=${PROBE_NQ:-100} ncu --profile-from-start off --clock-control none --set full --import-source on \
  -k "regex:$K" -s "$SKIP" -c 1 -o "$OUT" -f python profiles/graph_probe.py > "$OUT.log" 2>&1

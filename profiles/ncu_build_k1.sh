#!/bin/bash
# ncu --set full of K1 (k_summarise) on the c2 build, with and without the fine summary.
mkdir -p gpurun_out
python profiles/build_probe.py > gpurun_out/build_probe_plain.log 2>&1 || exit 1
TSG_NO_FINE=1 python profiles/build_probe.py >> gpurun_out/build_probe_plain.log 2>&1
ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:k_summarise -c 1 \
    -o gpurun_out/full_k1_fine -f python profiles/build_probe.py > gpurun_out/full_k1_fine.log 2>&1
TSG_NO_FINE=1 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:k_summarise -c 1 \
    -o gpurun_out/full_k1_nofine -f python profiles/build_probe.py > gpurun_out/full_k1_nofine.log 2>&1

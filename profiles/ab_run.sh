#!/bin/bash
# Generic A/B: the in-tree libtsgpu.so ("default") against variant builds
# (paper_2009_00786_b200/_variants/NAME.so, profiles/build_variant.sh), two alternating rounds of
# the c2 bench each. usage: bash profiles/ab_run.sh TAG NAME...   (outputs gpurun_out/ab_TAG_*.log)
tag=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
  python bench.py --no-cpu-baseline --no-other-configs --steps 20 --warmup 5 > gpurun_out/ab_${tag}_default_$r.log 2>&1
  for v in "$@"; do
    TSG_LIB_PATH=paper_2009_00786_b200/_variants/$v.so python bench.py --no-cpu-baseline --no-other-configs \
      --steps 20 --warmup 5 > gpurun_out/ab_${tag}_${v}_$r.log 2>&1
  done
done
python - "$tag" <<'PY'
import glob, json, sys
for f in sorted(glob.glob(f"gpurun_out/ab_{sys.argv[1]}_*.log")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f.split("/")[-1], "q/s", round(d["value"]), "e2e", round(d["e2e"]["value"]), "parity", d["parity"]["digest_equal"],
              d["roofline"]["per_kernel_us_per_query"], "build", d["build"]["phase_ms"])
    except Exception as e:
        print(f, "FAILED", e)
PY

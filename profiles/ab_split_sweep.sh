#!/bin/bash
# Sweep of the wave split (TSG_REFINE_SPLIT: runs / candidates below split x BSF go to wave 0 / A) on c2.
mkdir -p gpurun_out
for s in 0.2 0.25 0.3 0.35 0.4 0.5; do
  TSG_REFINE_SPLIT=$s python bench.py --no-cpu-baseline --no-other-configs --steps 20 --warmup 5 > gpurun_out/ab_split_$s.log 2>&1
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_split_*.log")):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f.split("/")[-1], round(d["value"]), d["parity"]["digest_equal"], d["roofline"]["per_slot_us_per_query"])
PY

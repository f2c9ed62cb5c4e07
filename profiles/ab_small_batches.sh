#!/bin/bash
# c5 small batches (sigma 0.01 / 0.1, batch 1 / 8 / 64) for the in-tree library and variant builds.
# usage: bash profiles/ab_small_batches.sh NAME...
for v in default "$@"; do
  L=""; [ $v != default ] && L=paper_2009_00786_b200/_variants/$v.so
  for b in 1 8 64; do for s in 0.01 0.1; do
    st=300; [ $b = 64 ] && st=40
    TSG_LIB_PATH=$L python bench.py --config c5 --batch $b --sigma $s --no-cpu-baseline --no-other-configs --steps $st --warmup 20 2>&1 | \
      python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith(chr(123))][-1]); print('$v batch $b sigma $s', round(d['value']), d['parity'].get('digest_equal') if d.get('parity') else None, d['roofline']['per_slot_us_per_query'])"
  done; done
done

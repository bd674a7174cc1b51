#!/bin/bash
# A/B of library builds / env knobs on ONE box (box-to-box variance is ~10%):
#   scripts/ab.sh "LABEL ENV=.. ENV=.." ...   each arg: a label then env assignments
for spec in "$@"; do
  set -- $spec
  label=$1; shift
  env "$@" python bench.py --steps 4 --warmup 3 --no-cpu --no-variants 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('%-28s %.3e ev/s  fwd %.2f  bwd %.2f ms' % ('$label', d['value'], r['fwd_ms'], r['bwd_ms']))"
done

#!/bin/bash
# A/B of library builds on ONE box with bench arguments:
#   scripts/ab_args.sh "BENCH ARGS" LABEL=LIB ...
args=$1; shift
for spec in "$@"; do
  label=${spec%%=*}; lib=${spec#*=}
  EQ_LIB_PATH=$lib python bench.py --steps 3 --warmup 3 --no-cpu --no-variants $args 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('%-8s %-60s %.3e ev/s  fwd %.2f  bwd %.2f ms' % ('$label', '$args', d['value'], r['fwd_ms'], r['bwd_ms']))"
done

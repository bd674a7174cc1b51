#!/bin/bash
# A/B of environment settings (and libraries) on ONE box with bench arguments:
#   scripts/ab_env.sh "BENCH ARGS" LABEL=LIB=ENV ...   (ENV: VAR=value, or "-" for none)
args=$1; shift
for spec in "$@"; do
  label=${spec%%=*}; rest=${spec#*=}; lib=${rest%%=*}; env=${rest#*=}
  [ "$env" = "-" ] && env=""
  env $env EQ_LIB_PATH=$lib python bench.py --steps 3 --warmup 3 --no-cpu --no-variants $args 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('%-8s %-40s %.3e ev/s  fwd %.2f  bwd %.2f ms' % ('$label', '$args', d['value'], r['fwd_ms'], r['bwd_ms']))"
done

#!/bin/bash
# Queue-variant sweep (BASELINE configs C2/C3/C4): one bench line per (config, kind).
# Usage: bash scripts/variant_sweep.sh OUT.jsonl [steps] [warmup]
OUT=${1:-gpurun_out/variants.jsonl}
K=${2:-3}
W=${3:-3}
: > "$OUT"
run() { python bench.py --steps $K --warmup $W --no-cpu --no-variants "$@" 2>>"${OUT%.jsonl}.err" | tail -1 >> "$OUT"; }
run --config C2 --trials 32 --kind ring
run --config C2 --trials 32 --kind binaryheap --capacity 64
run --config C2 --trials 32 --kind sortedarray --capacity 64
run --config C2 --trials 32 --kind fiforing --capacity 64 --delays 32,32
run --config C2 --trials 32 --kind ring --delays 32,32
run --config C3 --trials 16 --kind binaryheap --capacity 64
run --config C3 --trials 16 --kind sortedarray --capacity 64
# C4: memory-pressure regime, 1M neurons, delay <= 256, bounded queues drop
if [ -n "$C4" ]; then
  run --config C4 --trials 4 --kind ring
  run --config C4 --trials 4 --kind binaryheap --capacity 16
  run --config C4 --trials 4 --kind binaryheap --capacity 32
  run --config C4 --trials 4 --kind sortedarray --capacity 16
  run --config C4 --trials 4 --kind sortedarray --capacity 32
fi

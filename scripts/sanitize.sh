#!/bin/bash
# compute-sanitizer over small runs of every kernel family (memcheck, racecheck
# for shared-memory hazards, synccheck for barrier misuse).  Logs -> $OUT.
OUT=${1:-gpurun_out/sanitize}
mkdir -p $(dirname $OUT)
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_run.py > ${OUT}_${tool}.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Error|Invalid|Race)" ${OUT}_${tool}.log | head -5
done

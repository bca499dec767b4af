#!/bin/bash
# compute-sanitizer over every kernel family the solver selects (tools/sanitize_run.py).
# Usage: bash tools/sanitize.sh OUTDIR
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
for tool in memcheck racecheck synccheck initcheck; do
  for mode in graph-c1 chainw-c3 chainw-r-c1 dp-c1 fp32-c1 general; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 0 \
      python tools/sanitize_run.py $mode > "$out/${tool}_${mode}.log" 2>&1
    echo "$tool $mode rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' "$out/${tool}_${mode}.log" | tail -1)"
  done
done

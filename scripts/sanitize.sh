#!/bin/bash
# compute-sanitizer over the product kernels at small shapes (scripts/sanitize.py).
# Logs: gpurun_out/sanitize_<tool>.log ; summary line per tool at the end.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=${CS:-compute-sanitizer}
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      --target-processes all python scripts/sanitize.py ${SAN_CASES:-} > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done

#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck of the fit step kernels
# (one GPU; logs under gpurun_out/sanitize/, summarised into profiles/ by hand).
set -u
mkdir -p gpurun_out/sanitize
for case in ${CASES:-c1 c1mu c3 c5band}; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    timeout ${TMO:-900} compute-sanitizer --tool $tool $extra --print-limit 50 \
      python scripts/sanitize_step.py $case 2 > gpurun_out/sanitize/${case}_${tool}.log 2>&1
    echo "$case $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize/${case}_${tool}.log | tail -1)"
  done
done

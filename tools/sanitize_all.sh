#!/bin/bash
# compute-sanitizer over tools/sanitize_step.py: memcheck, racecheck, synccheck, initcheck
mkdir -p gpurun_out/sanitizer
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py > gpurun_out/sanitizer/r02_$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/sanitizer/r02_$t.log
done

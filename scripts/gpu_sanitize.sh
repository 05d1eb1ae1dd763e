#!/bin/bash
# compute-sanitizer over K1/K2/K3/K4 (scripts/sanitize_cases.py); logs to
# gpurun_out/sanitize/.  Usage (on the GPU box): bash scripts/gpu_sanitize.sh
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in cfg1 cfg2 weighted; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    log=gpurun_out/sanitize/${tool}_${case}.log
    echo "== $tool $case" | tee -a gpurun_out/sanitize/summary.txt
    timeout 900 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize_cases.py $case > $log 2>&1
    rc=$?
    echo "rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' $log | tr '\n' ' ')" | tee -a gpurun_out/sanitize/summary.txt
  done
done

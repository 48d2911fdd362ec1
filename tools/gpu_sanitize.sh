#!/bin/bash
# compute-sanitizer over the hot path (verdict r1 item 10). Summaries -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for w in ${WORKLOADS:-c1 chain wide}; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize.py $w \
      > gpurun_out/sanitize_${tool}_${w}.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_${tool}_${w}.log
  done
done

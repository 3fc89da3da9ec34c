#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py; logs to gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  arg=""
  [ "$tool" = racecheck ] && arg=small
  [ "$tool" = initcheck ] && arg=small
  timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py $arg \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
done

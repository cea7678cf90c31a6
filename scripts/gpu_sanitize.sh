#!/bin/bash
# compute-sanitizer over scripts/sanitize.py: memcheck, racecheck, synccheck (one tool per pass)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py \
     > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.txt
done

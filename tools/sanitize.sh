#!/bin/bash
# compute-sanitizer over every device path (tools/sanitize_cases.py); summaries -> gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.log
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.log
done

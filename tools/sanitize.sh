#!/usr/bin/env bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_driver.py
# (SURVEY.md §5).  Summaries -> gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -n 3 gpurun_out/sanitize_*.log

#!/bin/bash
# compute-sanitizer passes over tools/sanitize_target.py; logs in gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_target.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.log
  tail -3 gpurun_out/sanitize_$tool.log
done

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
# (run under gpurun on one GPU); logs in gpurun_out/sanitize_*.log
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|ok$" gpurun_out/sanitize_$tool.log | tail -6
done

#!/bin/bash
# compute-sanitizer tiers over tools/sanitize_driver.py (run under gpurun).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 3 --target-processes all \
    python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|done' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done

#!/bin/bash
# compute-sanitizer over scripts/sanitize_smoke.py (outputs under gpurun_out/); each tool bounded
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
    python scripts/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool=$?"; tail -3 gpurun_out/sanitize_$tool.log
done

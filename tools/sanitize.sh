#!/bin/bash
# compute-sanitizer over every kernel (run under gpurun):
#   gpurun -- 'bash tools/sanitize.sh'  -> gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool cases rc=$?"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python -m pytest tests/test_step_api.py -m gpu -q -x -k "select or eviction" > gpurun_out/sanitize_${tool}_step.log 2>&1
  echo "$tool step-api rc=$?"
done

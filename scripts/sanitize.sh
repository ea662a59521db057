#!/bin/bash
# compute-sanitizer over every kernel path (tools/sanitize_cases.py); summaries in gpurun_out/.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.txt
done

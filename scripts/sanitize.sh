#!/bin/bash
# compute-sanitizer over small products on both paths; summaries into gpurun_out/.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize_small" gpurun_out/sanitize_$tool.txt >> gpurun_out/sanitize_summary.txt
done

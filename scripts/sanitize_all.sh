#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py, one tool at a time
mkdir -p gpurun_out
timeout 600 python scripts/sanitize_run.py > gpurun_out/san_plain.txt 2>&1
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 2000 python scripts/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok" gpurun_out/san_$tool.txt >> gpurun_out/san_summary.txt
done

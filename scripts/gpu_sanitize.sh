#!/bin/bash
mkdir -p gpurun_out/san
python scripts/sanitize_cases.py > gpurun_out/san/plain.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log >> gpurun_out/san/summary.txt
done

#!/bin/bash
# compute-sanitizer over every kernel (scripts/sanitize_cases.py); summary in gpurun_out/san/summary.txt
mkdir -p gpurun_out/san
rm -f gpurun_out/san/summary.txt
python scripts/sanitize_cases.py > gpurun_out/san/plain.log 2>&1
echo "plain rc=$?" >> gpurun_out/san/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  if [ $tool = synccheck ]; then extra="--num-cuda-barriers 65536"; fi
  timeout 900 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log >> gpurun_out/san/summary.txt
done
cat gpurun_out/san/summary.txt

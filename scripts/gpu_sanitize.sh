#!/bin/bash
# compute-sanitizer over every kernel family on tiny shapes (scripts/sanitize.py)
mkdir -p gpurun_out
python paper_2312_12456_b200/build.py > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_$tool.txt | tail -1)"
done

#!/bin/bash
# full GPU pass: tests, smoke, c4 bench + reference arm, ncu launch list + full capture (summarised),
# layer trace, compute-sanitizer, secondary bench lines
python paper_2312_12456_b200/build.py > /dev/null
./scripts/gpu_final.sh
./scripts/gpu_sanitize.sh
bash scripts/gpu_bench_lines.sh

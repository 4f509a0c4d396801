#!/bin/bash
# round-end style check: tests, smoke, bench lines, reference arm, ncu launch list + one full capture
# (summarised here; the .ncu-rep files are deleted so gpurun_out/ stays under the copy-back limit)
./scripts/gpu_check.sh
python scripts/ncu_summary.py launches gpurun_out/launches_c4.csv > gpurun_out/launches_c4.txt 2>&1
python scripts/ncu_summary.py full gpurun_out/prof_stack_c4.ncu-rep > gpurun_out/ncu_full_c4.txt 2>&1
ncu -i gpurun_out/prof_stack_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/src_c4.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
timeout 300 python scripts/trace_layer.py --config c4 --stack > gpurun_out/trace_c4_stack.json 2>&1
du -sh gpurun_out; ls gpurun_out

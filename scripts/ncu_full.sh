#!/bin/bash
# one ncu --set full capture (with source) of the c4 stack kernel (8 layers), then the source page as CSV
mkdir -p gpurun_out
python paper_2312_12456_b200/build.py > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer -s 2 -c 1 -o gpurun_out/prof_${TAG:-x} -f \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --layers ${LAYERS:-8} > gpurun_out/ncu_full_${TAG:-x}.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_${TAG:-x}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG:-x}.csv 2> gpurun_out/src_${TAG:-x}.err; echo src=$?
ls -la gpurun_out/ | tail -5

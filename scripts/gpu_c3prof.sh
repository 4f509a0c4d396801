python paper_2312_12456_b200/build.py > /dev/null
for b in 4 8 16; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_c3b$b.csv python bench.py --config c3 --batch $b --layers 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-phases > gpurun_out/ncu_c3b$b.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py launches gpurun_out/launches_c3b$b.csv 2>&1 | head -16
done

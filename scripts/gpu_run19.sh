python paper_2312_12456_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_c3b16.csv python bench.py --config c3 --batch 16 --layers 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-phases > gpurun_out/ncu_c3b16.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py launches gpurun_out/launches_c3b16.csv 2>&1 | head -14
LINES="c3:16 c3:32" bash scripts/gpu_bench_lines.sh

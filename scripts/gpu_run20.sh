python paper_2312_12456_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
LINES="c4q4:1 c3:16" bash scripts/gpu_bench_lines.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_up_tc -s 3 -c 1 -o gpurun_out/prof_uptc -f python bench.py --config c3 --batch 16 --layers 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-phases > gpurun_out/ncu_uptc.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py full gpurun_out/prof_uptc.ncu-rep > gpurun_out/ncu_uptc.txt 2>&1; head -30 gpurun_out/ncu_uptc.txt
ncu -i gpurun_out/prof_uptc.ncu-rep --page details --csv > gpurun_out/uptc_details.csv 2>/dev/null; rm -f gpurun_out/prof_uptc.ncu-rep

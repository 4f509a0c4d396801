#!/bin/bash
# GPU check: parity tests, smoke, bench lines, ncu launch list + one full capture of the stack kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo b4=$?; tail -2 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --config c2 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?; cat gpurun_out/bench_c2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bref=$?; cat gpurun_out/bench_ref.json
if [ "${PI_NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer -s 2 -c 1 -o gpurun_out/prof_stack_c4 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --layers 8 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi

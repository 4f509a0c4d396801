#!/bin/bash
# quick GPU iteration: parity tests (fused + per-step paths), phase traces, bench lines
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
for c in c4 c2 c5 c1; do timeout 300 python scripts/trace_layer.py --config $c > gpurun_out/trace_$c.json 2>&1; cat gpurun_out/trace_$c.json; done
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo b4=$?; tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --config c2 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?; cat gpurun_out/bench_c2.json

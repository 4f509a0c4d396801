#!/bin/bash
# one GPU iteration: parity tests (TESTS=0 skips; PYTEST_K selects), c4 stack trace, c4 bench line
mkdir -p gpurun_out
python paper_2312_12456_b200/build.py > /dev/null
if [ "${TESTS:-1}" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
fi
timeout 300 python scripts/trace_layer.py --config ${CFG:-c4} --stack ${TRACE_ARGS} > gpurun_out/trace.json 2>&1
python -c "
import json; j=json.load(open('gpurun_out/trace.json')); print('trace'); print(' mean', j['phases_us_mean_over_ctas']); print(' max ', j['phases_us_max_over_ctas'])" || tail -5 gpurun_out/trace.json
timeout 900 python bench.py --config ${CFG:-c4} --steps 30 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; j=json.load(open('gpurun_out/bench.json')); print('bench', j['value'], j['ms_per_step'], j['roofline']['frac'], j['e2e']['value']); print(json.dumps(j.get('phases_us'))); print(json.dumps(j.get('cpu_baseline')))" || tail -20 gpurun_out/bench.err

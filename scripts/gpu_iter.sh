#!/bin/bash
# one GPU iteration: parity tests, then per knob setting: c4 stack trace + c4 bench line (no CPU baseline)
mkdir -p gpurun_out
python paper_2312_12456_b200/build.py > /dev/null
if [ "${TESTS:-1}" = "1" ]; then
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
fi
for k in ${KNOBS:-0}; do
PI_FUSED_KNOBS=$k timeout 300 python scripts/trace_layer.py --config ${CFG:-c4} --stack > gpurun_out/trace_k$k.json 2>&1
python -c "
import json; j=json.load(open('gpurun_out/trace_k$k.json')); print('trace knobs=$k'); print(' mean', j['phases_us_mean_over_ctas']); print(' max ', j['phases_us_max_over_ctas'])" || tail -5 gpurun_out/trace_k$k.json

PI_FUSED_KNOBS=$k timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_k$k.json 2> gpurun_out/bench_c4_k$k.err
python -c "
import json; j=json.load(open('gpurun_out/bench_c4_k$k.json')); print('bench knobs=$k', j['value'], j['ms_per_step'], j['roofline']['frac'], j['e2e']['value'])" || tail -5 gpurun_out/bench_c4_k$k.err
done

#!/bin/bash
# final: every GPU test, smoke, one c4 bench line (driver-style), all logs under gpurun_out/final2
mkdir -p gpurun_out/final2
python paper_2312_12456_b200/build.py > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/final2/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/final2/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/final2/bench_c4_default.json 2> gpurun_out/final2/bench_c4_default.err; echo bench=$?
python -c "
import json; j=json.load(open('gpurun_out/final2/bench_c4_default.json')); print('c4', round(j['value'],1), round(j['ms_per_step'],4), j['roofline']['frac'], j['e2e']['value'], j['gpu_launches'], j['clocks'])"

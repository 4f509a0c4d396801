#!/bin/bash
# parity tests (all GPU tests) + grouped lines + c4 / c4-int4 / c2 lines
mkdir -p gpurun_out/it
python paper_2312_12456_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/it/pytest.log 2>&1; echo pytest=$?; tail -4 gpurun_out/it/pytest.log
LINES="${GLINES:-c1:2 c1:4 c2:8 c2:37}" bash scripts/gpu_group.sh 2>&1 | grep -E "pg|pytest"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/it/c4.json 2> gpurun_out/it/c4.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --q4 --hot-freq 0 > gpurun_out/it/c4q4.json 2> gpurun_out/it/c4q4.err
timeout 600 python bench.py --config c2 --no-group --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/it/c2s.json 2> gpurun_out/it/c2s.err
for f in c4 c4q4 c2s; do python -c "
import json; j=json.load(open('gpurun_out/it/$f.json')); print('$f', round(j['value'],1), round(j['ms_per_step'],4), j['roofline']['frac'], j.get('phases_us'))" || tail -3 gpurun_out/it/$f.err; done

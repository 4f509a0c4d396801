#!/bin/bash
mkdir -p gpurun_out/it3
python paper_2312_12456_b200/build.py > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_gpu_multiproc.py -q -x -p no:cacheprovider > gpurun_out/it3/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/it3/pytest.log
for a in "c4 1" "c3 1" "c3 2"; do set -- $a
timeout 600 python bench.py --config $1 --batch $2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/it3/$1_b$2.json 2> gpurun_out/it3/$1_b$2.err
python -c "
import json; j=json.load(open('gpurun_out/it3/$1_b$2.json')); print('$1 b$2', round(j['value'],1), round(j['ms_per_step'],4), j['roofline']['frac'], j.get('phases_us'))" || tail -3 gpurun_out/it3/$1_b$2.err
done

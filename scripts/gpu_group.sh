#!/bin/bash
# grouped launch: parity tests and c1 / c2 bench lines over group sizes
mkdir -p gpurun_out/group
python paper_2312_12456_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_group.py -q -x -p no:cacheprovider > gpurun_out/group/pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/group/pytest.log
for cfg_pg in ${LINES:-c1:1 c1:2 c1:4 c2:4 c2:8 c2:12}; do
  c=${cfg_pg%%:*}; pg=${cfg_pg##*:}
  timeout 600 python bench.py --config $c --group-ctas $pg --steps 30 --warmup 5 --no-cpu-baseline ${EXTRA} > gpurun_out/group/${c}_pg$pg.json 2> gpurun_out/group/${c}_pg$pg.err
  python -c "
import json; j=json.load(open('gpurun_out/group/${c}_pg$pg.json')); print('$c pg $pg', round(j['value']), 'tok/s', round(j['ms_per_step'],3), 'ms frac', j['roofline']['frac'], 'act', j['config']['realised_activity'], 'e2e', round(j['e2e']['value']))" || tail -5 gpurun_out/group/${c}_pg$pg.err
done

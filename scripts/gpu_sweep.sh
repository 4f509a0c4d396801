#!/bin/bash
# c4 bench sweep over one bench flag: FLAG="--l2-prefetch" VALS="0 2 4 8"
python paper_2312_12456_b200/build.py > /dev/null
for v in ${VALS}; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e ${EXTRA} ${FLAG} $v > gpurun_out/sweep_$v.json 2> gpurun_out/sweep_$v.err
  python -c "
import json; j=json.load(open('gpurun_out/sweep_$v.json')); ph=j.get('phases_us') or {}
print('${FLAG} $v', round(j['value'],1), round(j['ms_per_step'],4), j['roofline']['frac'], 'FFN', ph.get('FFN up+down (a4+a5)'), 'P2', ph.get('P2 + threshold (a2)'), 'layer', ph.get('layer_total'))" || tail -5 gpurun_out/sweep_$v.err
done

#!/bin/bash
# c4 bench with the speculative prefix off and on (17-warp kernel), plus the traces
python paper_2312_12456_b200/build.py > /dev/null
for s in 0 0.99; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --spec-freq $s --hot-freq 0.99 > gpurun_out/bench_spec$s.json 2> gpurun_out/bench_spec$s.err
  python -c "
import json; j=json.load(open('gpurun_out/bench_spec$s.json')); print('spec $s', round(j['value'],1), round(j['ms_per_step'],4), j['roofline']['frac']); print(json.dumps(j.get('phases_us')))" || tail -5 gpurun_out/bench_spec$s.err
done

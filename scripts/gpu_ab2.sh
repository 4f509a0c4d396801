#!/bin/bash
AB_CFGS="c4:1 c3:1" bash scripts/gpu_ab.sh
for cap in 512 768 1024; do for hf in 0.99 0.9; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --hot-cap $cap --hot-freq $hf > gpurun_out/ab/cap_${cap}_$hf.json 2>&1
python -c "
import json; j=json.load(open('gpurun_out/ab/cap_${cap}_$hf.json')); ph=j.get('phases_us') or {}; print('cap $cap hf $hf', round(j['ms_per_step'],4), j['roofline']['frac'], {k: ph.get(k) for k in ('P2 + threshold (a2)','compaction (a3)','FFN up+down (a4+a5)','layer_total')})"
done; done

#!/bin/bash
for dbg in 0 1 2 4 3; do
  PI_FUSED_DEBUG=$dbg timeout 300 python scripts/trace_layer.py --config ${1:-c4} > gpurun_out/trace_dbg$dbg.json 2>&1
  python -c "
import json
j=json.load(open('gpurun_out/trace_dbg$dbg.json'))
print('dbg=$dbg', j['ideal_us_at_peak'], {k: v for k, v in j['phases_us_mean_over_ctas'].items()})
print('   ready', j['cta0_stage_ready_us'])
"
done

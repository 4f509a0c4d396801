#!/bin/bash
# bench lines for the secondary workloads: c3 at B = 1..32 (batched tensor-core path
# above 8), c4 with INT4 rows, c4 with ILP placement, c2 / c1 single layers.  One JSON line each.
mkdir -p gpurun_out/lines
python paper_2312_12456_b200/build.py > /dev/null
run() {  # name, args...
  local n=$1; shift
  timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline "$@" > gpurun_out/lines/$n.json 2> gpurun_out/lines/$n.err
  python -c "
import json,sys
try:
    j=json.load(open('gpurun_out/lines/$n.json'))
    print('$n', round(j['value'],1), 'tok/s', round(j['ms_per_step'],3), 'ms', 'frac', j['roofline']['frac'], 'step_frac', j['roofline']['step_frac'], 'act', j['config'].get('realised_activity'))
except Exception as e:
    print('$n FAILED', e); print(open('gpurun_out/lines/$n.err').read()[-1500:])"
}
LINES=${LINES:-c3:1 c3:2 c3:4 c3:8 c3:16 c3:32 c4q4:1 c2:1 c1:1}
for cfgb in $LINES; do
  c=${cfgb%%:*}; bb=${cfgb##*:}
  case $c in
    c4q4) run c4_q4_b$bb --config c4 --batch $bb --q4 --hot-freq 0 ;;
    c4ilp) run c4_ilp_b$bb --config c4 --batch $bb --placement ilp ;;
    *) run ${c}_b$bb --config $c --batch $bb ;;
  esac
done

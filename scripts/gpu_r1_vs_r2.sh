#!/bin/bash
# same-box comparison of the round-1 build (worktree _r1 at 4f49af5, its own bench.py) and this build
python paper_2312_12456_b200/build.py > /dev/null
for rep in 1 2; do
  (cd _r1 && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/r1.json 2>/tmp/r1.err; python -c "
import json; j=json.load(open('/tmp/r1.json')); print('round-1 build', round(j['ms_per_step'],4), j['roofline']['frac'], j['value'])" || tail -3 /tmp/r1.err)
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/r2.json 2>/tmp/r2.err; python -c "
import json; j=json.load(open('/tmp/r2.json')); print('round-2 build', round(j['ms_per_step'],4), j['roofline']['frac'], j['value'])" || tail -3 /tmp/r2.err
done

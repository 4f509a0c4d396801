#!/bin/bash
# same-box c4 bench of several builds (each worktree runs its own bench.py); dirs as arguments
for rep in ${REPS:-1 2}; do
for d in "$@"; do
  (cd $d && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/bb.json 2>/tmp/bb.err; python -c "
import json; j=json.load(open('/tmp/bb.json')); ph=j.get('phases_us') or {}; print('$d', round(j['ms_per_step'],4), j['roofline']['frac'], {k: ph.get(k) for k in ('P1 (a1)','P2 + threshold (a2)','compaction (a3)','FFN up+down (a4+a5)','grid barrier 3','reduction of partials')})" || tail -3 /tmp/bb.err)
done; done

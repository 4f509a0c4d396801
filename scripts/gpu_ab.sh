#!/bin/bash
# A/B on one box: paper_2312_12456_b200/libpi_base.so (A) vs the tree's libpi.so (B), alternating
mkdir -p gpurun_out/ab
cp paper_2312_12456_b200/libpi.so paper_2312_12456_b200/libpi_new.so
run() { # tag lib cfg b
  cp paper_2312_12456_b200/$2 paper_2312_12456_b200/libpi.so
  timeout 600 python bench.py --config $3 --batch $4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab/$1.json 2> gpurun_out/ab/$1.err
  python -c "
import json; j=json.load(open('gpurun_out/ab/$1.json')); ph=j.get('phases_us') or {}; print('$1', round(j['ms_per_step'],4), j['roofline']['frac'], {k: ph.get(k) for k in ('P1 (a1)','compaction (a3)','FFN up+down (a4+a5)','layer_total')})" || tail -3 gpurun_out/ab/$1.err
}
for rep in 1 2; do
  for cb in ${AB_CFGS:-c4:1 c3:1}; do c=${cb%%:*}; b=${cb##*:}
    run A_${c}_b${b}_$rep libpi_base.so $c $b
    run B_${c}_b${b}_$rep libpi_new.so $c $b
  done
done
cp paper_2312_12456_b200/libpi_new.so paper_2312_12456_b200/libpi.so

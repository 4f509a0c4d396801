python paper_2312_12456_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_group.py -q -x -p no:cacheprovider 2>&1 | tail -2
for f in 0 1 2; do for cfg_pg in c2:8 c1:2 c2:4; do c=${cfg_pg%%:*}; pg=${cfg_pg##*:}
timeout 600 python bench.py --config $c --group-ctas $pg --group-defer $f --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/gd_${c}_$pg_$f.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/gd_${c}_$pg_$f.json')); print('$c pg $pg defer $f', round(j['value']), round(j['ms_per_step'],3), j['roofline']['frac'])" 2>&1 | tail -1; done; done

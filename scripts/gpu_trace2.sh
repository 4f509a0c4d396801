python paper_2312_12456_b200/build.py > /dev/null
timeout 300 python scripts/trace_layer.py --config c4 --stack --q4 > gpurun_out/trace_c4q4.json 2>&1
python -c "
import json; j=json.load(open('gpurun_out/trace_c4q4.json')); print('c4q4 mean', j['phases_us_mean_over_ctas']); print('ready', j['cta0_stage_ready_us']); print('issue', j['cta0_stage_issue_us'])" || tail -5 gpurun_out/trace_c4q4.json
for a in "c1 2 74 3" "c2 8 18 3"; do timeout 300 python scripts/dbg/group_trace.py $a 2>&1 | tail -4 | cut -c1-1500; done
for cfg_pg in c1:2 c2:8; do c=${cfg_pg%%:*}; pg=${cfg_pg##*:}; timeout 600 python bench.py --config $c --group-ctas $pg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/g_$c.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/g_$c.json')); print('$c pg $pg', round(j['value']), round(j['ms_per_step'],3), j['roofline']['frac'])"; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --q4 --hot-freq 0 > gpurun_out/c4q4.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/c4q4.json')); print('c4q4', round(j['value']), round(j['ms_per_step'],3), j['roofline']['frac'], j['phases_us'])"

#!/bin/bash
# round-2 final pass: tests, smoke, c4 bench + reference arm, ncu launch list + full capture, trace,
# secondary lines (grouped c1/c2, c3 B = 1..32, c4 INT4, c4 activity 5 / 20 %, c4 predictor rank 1472)
mkdir -p gpurun_out/final/lines
rm -f paper_2312_12456_b200/libpi_base.so paper_2312_12456_b200/libpi_new.so
python paper_2312_12456_b200/build.py > /dev/null
nvidia-smi > gpurun_out/final/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/final/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err; echo b4=$?
python -c "
import json; j=json.load(open('gpurun_out/final/bench_c4.json')); print('c4', j['value'], j['ms_per_step'], j['roofline']['frac'], j['e2e']['value'], j['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo bref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/final/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_launch.log 2>&1; echo ncu1=$?
python scripts/ncu_summary.py launches gpurun_out/final/launches_c4.csv > gpurun_out/final/launches_c4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer -s 2 -c 1 -o gpurun_out/final/prof_stack_c4 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --layers 8 > gpurun_out/final/ncu_full.log 2>&1; echo ncu2=$?
python scripts/ncu_summary.py full gpurun_out/final/prof_stack_c4.ncu-rep > gpurun_out/final/ncu_full_c4.txt 2>&1
rm -f gpurun_out/final/*.ncu-rep
timeout 300 python scripts/trace_layer.py --config c4 --stack --hot-freq 0.99 > gpurun_out/final/trace_c4_stack.json 2>&1
run() {  # name, args...
  local n=$1; shift
  timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline "$@" > gpurun_out/final/lines/$n.json 2> gpurun_out/final/lines/$n.err
  python -c "
import json
j=json.load(open('gpurun_out/final/lines/$n.json'))
print('$n', round(j['value'],1), 'tok/s', round(j['ms_per_step'],4), 'ms frac', j['roofline']['frac'], 'act', j['config'].get('realised_activity'))" || tail -3 gpurun_out/final/lines/$n.err
}
run c1_grouped --config c1
run c2_grouped --config c2
run c2_single --config c2 --no-group
for b in 1 2 4 8 16 32; do run c3_b$b --config c3 --batch $b; done
run c4_q4 --q4 --hot-freq 0
run c4_act05 --mean-act 0.05
run c4_act20 --mean-act 0.20
run c4_rank1472 --rank 1472
run c4_b2 --batch 2
ls gpurun_out/final

timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
AB_CFGS="c4:1 c3:4 c3:8" bash scripts/gpu_ab.sh
for lib in libpi_base.so libpi_new.so; do cp paper_2312_12456_b200/$lib paper_2312_12456_b200/libpi.so
timeout 600 python bench.py --config c1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab/c1_$lib.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/ab/c1_$lib.json')); print('c1 $lib', round(j['ms_per_step'],4), j['roofline']['frac'])"
done
cp paper_2312_12456_b200/libpi_new.so paper_2312_12456_b200/libpi.so

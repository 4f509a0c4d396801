timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
TESTS=0 BENCH_ARGS="--spec-freq 0" bash scripts/gpu_iter.sh
mv gpurun_out/bench.json gpurun_out/bench_nospec.json
TESTS=0 TRACE_ARGS="--spec-freq 0.99 --hot-freq 0.9" bash scripts/gpu_iter.sh
python -c "import json;s=open('gpurun_out/trace.json').read();j=json.loads(s[s.index('{'):]);print(j['phases_us_mean_over_ctas'])"

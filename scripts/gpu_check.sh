set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --config c2 --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo b2=$?; tail -3 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo b4=$?; tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json

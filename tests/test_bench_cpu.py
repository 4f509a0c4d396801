"""bench.py's host-side contract on CPU: --gpus N (no torchrun env) re-launches itself with N
ranks and prints ONE JSON line with n_gpus = N (the --dry-run plumbing check: gloo, the per-layer
all-reduce, max-over-ranks timing); --impl reference prints the oracle arm's line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.timeout(600)
def test_bench_spawns_n_ranks_dry_run():
    j = _run(["--gpus", "2", "--dry-run", "--steps", "3", "--warmup", "3", "--config", "c4", "--layers", "4"])
    assert j["n_gpus"] == 2 and j["dry_run"] is True and j["steps"] == 3 and j["warmup"] == 3
    assert j["value"] > 0 and j["ms_per_step"] > 0
    assert j["config"]["parallelism"].startswith("neuron-sharded x2")


@pytest.mark.timeout(600)
def test_bench_reference_arm_line():
    j = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"])
    assert j["impl"] == "reference" and j["unit"] == "tokens/s" and j["value"] > 0
    assert j["step"] == "one token-batch through one layer"
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0

#!/usr/bin/env python
"""bench.py -- sparse-FFN decode tokens/s and % of the HBM roofline on activated-neuron bytes.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl pi|reference]

One step = one decode token (batch B) through every layer of the workload: the whole hot
path of SURVEY.md 8(a) (predictor -> mask -> compaction -> row-sparse up -> column-sparse
down [-> NCCL all-reduce for N > 1]).  Default workload: configs[3] of BASELINE.json, the
Falcon-40B-ReLU FFN stack (d 8192, m 32768, 60 layers, predictor rank 512), the config the
metric's "1/2/4/8 B200" refers to; it fits one GPU (64 GB of FFN weights), so at N = 1 it is
the single-GPU workload and at N > 1 it is neuron-sharded across ranks (strong scaling).
``--config c2`` runs the single OPT-6.7B layer (rotated over 16 copies to defeat L2).

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "sparse-FFN decode tokens/s and % HBM roofline (active bytes) at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None, help="override the layer count (debug only)")
    ap.add_argument("--copies", type=int, default=16, help="layer copies rotated for single-layer configs")
    ap.add_argument("--impl", default="pi", choices=["pi", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=15.0, help="CPU budget of the oracle baseline")
    ap.add_argument("--hot-freq", type=float, default=0.99,
                    help="hot neurons (Insight-1): the fused kernel L2-prefetches the rows of up to PI_HOT_CAP "
                         "(default 512) neurons per layer whose profiled activation frequency is >= this, "
                         "while the layer synchronises after phase 2 (<= 0 disables; c4: 2.22 vs 2.30 ms/step)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.dev = dev_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# CPU oracle baseline (TEST/BASELINE leg only: the one place bench.py runs oracle/)
# ---------------------------------------------------------------------------
def oracle_baseline(cfg, seed, n_layers_total, B, seconds, device):
    """Time oracle predict -> compact -> sparse_ffn on host cores for a bounded sample."""
    from oracle import ffn as O
    from paper_2312_12456_b200 import gen

    k = 2 if n_layers_total > 1 else 1
    t_layer = []
    samples = 0
    t_start = time.perf_counter()
    for l in range(k):
        w = gen.make_layer(cfg, layer=l, seed=seed, device=device)
        f = lambda t: None if t is None else t.float().cpu().numpy()  # noqa: E731
        W = {kk: f(v) for kk, v in w.tensors().items()}
        del w
        tok = 0
        while True:
            x = gen.tokens(B, cfg.d, seed=seed + 99, step=tok, device="cpu").numpy().astype(np.float64)
            t0 = time.perf_counter()
            xo = O.rms_normalize(x) if cfg.rmsnorm else x
            mask, _ = O.predict(xo, W["p_w1"], W["p_b1"], W["p_w2"], W["p_b2"], 0.0)
            ids = O.compact(mask)
            O.sparse_ffn(xo, ids, mask, W["w_up"], W["b_up"], W["w_gate"], W["w_down"], W["b_down"], cfg.act)
            t_layer.append(time.perf_counter() - t0)
            tok += 1
            samples += 1
            if sum(t_layer) > seconds * (l + 1) / k or tok >= 64:
                break
        del W
    per_layer = float(np.mean(t_layer))
    value = B / (per_layer * n_layers_total)
    return {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle",
            "sample": f"{samples} (token-batch, layer) pairs over layers 0..{k - 1} of {n_layers_total}, "
                      f"B={B}; full-stack time extrapolated x{n_layers_total}; numpy fp64 single-threaded "
                      f"(elementwise ops, no BLAS in the timed path); weight generation and host copies untimed",
            "seconds": round(time.perf_counter() - t_start, 1)}


def run_reference(args, cfg, B, n_layers):
    """--impl reference: the oracle as it stands on the host cores, same config/metric/unit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ffn as O
    from paper_2312_12456_b200 import gen

    k = min(2, n_layers)
    Ws = []
    for l in range(k):
        w = gen.make_layer(cfg, layer=l, seed=args.seed, device="cpu")
        f = lambda t: None if t is None else t.float().numpy()  # noqa: E731
        Ws.append({kk: f(v) for kk, v in w.tensors().items()})
        del w

    def one(step):
        W = Ws[step % k]
        x = gen.tokens(B, cfg.d, seed=args.seed, step=step, device="cpu").numpy().astype(np.float64)
        t0 = time.perf_counter()
        xo = O.rms_normalize(x) if cfg.rmsnorm else x
        mask, _ = O.predict(xo, W["p_w1"], W["p_b1"], W["p_w2"], W["p_b2"], 0.0)
        ids = O.compact(mask)
        O.sparse_ffn(xo, ids, mask, W["w_up"], W["b_up"], W["w_gate"], W["w_down"], W["b_down"], cfg.act)
        return time.perf_counter() - t0

    for i in range(args.warmup):
        one(i)
    ts = [one(args.warmup + i) for i in range(args.steps)]
    per_layer = float(np.mean(ts))
    ms_step = per_layer * n_layers * 1e3
    value = B / (per_layer * n_layers)
    sample = (f"each step = one token-batch (B={B}) through one of layers 0..{k - 1}; per-step time extrapolated "
              f"x{n_layers} layers; numpy fp64, single thread")
    out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference", "config": workload_config(cfg, B, n_layers, args.gpus, hot_freq=args.hot_freq),
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def workload_config(cfg, B, n_layers, N, extra=None, hot_freq=0.0):
    c = {"workload": f"{cfg.name}: {cfg.desc}", "d": cfg.d, "ffn": cfg.m, "predictor_rank": cfg.r,
         "layers": n_layers, "batch": B, "act": cfg.act, "weights": cfg.dtype, "activations": "fp32",
         "mean_activity_target": 0.10, "mask_mode": "P (predictor-generated, planted b2)",
         "parallelism": "single GPU" if N == 1 else f"neuron-sharded x{N} (pi_partition) + NCCL all-reduce",
         "hot_neurons": ("L2 prefetch of <= %s neurons/layer with profiled frequency >= %g" %
                         (os.environ.get("PI_HOT_CAP", "512"), hot_freq)) if hot_freq > 0 else "off"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------------------
def main():
    args = parse()
    from paper_2312_12456_b200 import gen

    cfg = gen.CONFIGS[args.config]
    B = args.batch or cfg.batch
    n_layers = args.layers or cfg.layers
    if args.impl == "reference":
        run_reference(args, cfg, B, n_layers)
        return

    import torch.distributed as dist
    from paper_2312_12456_b200 import pi
    from paper_2312_12456_b200.stack import algorithmic_bytes, build_stack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    # ---- build the workload (weights random-init with the config's architecture) ----
    single = n_layers == 1
    copies = args.copies if single else 1
    stacks = []
    for c in range(copies):
        st, _ = build_stack(cfg, n_layers=n_layers, rank=rank, world=world, seed=args.seed + 1000 * c,
                            device=dev, max_batch=B, group=group,
                            hot_freq=args.hot_freq if args.hot_freq > 0 else None)
        stacks.append(st)
    d = cfg.d
    T = args.warmup + args.steps
    xs = torch.stack([gen.tokens(B, d, seed=args.seed + 7, step=i, device=dev) for i in range(T)])
    y = torch.empty(B, d, device=dev)
    bufs = [torch.empty(B, d, device=dev) for _ in range(2)]
    nbuf = torch.zeros(T, n_layers, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step(i, record_n=True):
        st = stacks[i % copies]
        st.step(xs[i], y, nbuf[i] if record_n else None, bufs)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up, then EXACTLY K timed steps ----
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for k in range(args.steps):
        step(args.warmup + k)
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    per_step = np.array([evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)])
    total_ms = evs[0].elapsed_time(evs[-1])
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = B * args.steps / (total_ms / 1e3)          # tokens of the whole job (all ranks share them)

    # ---- realised activity and algorithmic bytes (from the counts written during the timed steps) ----
    n_host = nbuf.cpu().numpy()[args.warmup:]
    metas = stacks[0].metas
    bytes_step = np.array([[algorithmic_bytes(metas[l], int(n_host[k, l]), B) for l in range(n_layers)]
                           for k in range(args.steps)])
    realised = float(n_host.mean() / metas[0].m_local)

    # ---- dominant kernel: per-launch durations with CUDA events on the launching stream ----
    # world 1: the stack kernel (one launch = one step through every layer);
    # world > 1: the per-layer fused kernel (launches separated by the NCCL all-reduce)
    prof_steps = min(args.steps, 10)
    kt, kb = [], []
    for k in range(prof_steps):
        i = args.warmup + k
        st = stacks[i % copies]
        if world == 1:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st.step(xs[i], y, None, bufs)
            e1.record(stream)
            torch.cuda.synchronize()
            kt.append(e0.elapsed_time(e1) / 1e3)
            kb.append(float(bytes_step[k].sum()))
            continue
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_layers)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_layers)]
        cur = xs[i]
        for l, L in enumerate(st.layers):
            dst = bufs[l & 1]
            e0[l].record(stream)
            L.forward(cur, dst)
            e1[l].record(stream)
            dist.all_reduce(dst)
            cur = dst
        torch.cuda.synchronize()
        for l in range(n_layers):
            kt.append(e0[l].elapsed_time(e1[l]) / 1e3)
            kb.append(algorithmic_bytes(metas[l], int(n_host[k, l]), B))
    launch_s = float(np.mean(kt))
    bytes_launch = float(np.mean(kb))
    peak, peak_src = hbm_peak()
    achieved = bytes_launch / launch_s / 1e9
    launches_per_layer = int(stacks[0].layers[0].info.launches_per_forward)
    kname = ("k_layer x%d layers in one persistent launch (pi_stack_run)" % n_layers) if world == 1 and \
        launches_per_layer == 1 else "pi_layer_forward (%d launch(es) per layer)" % launches_per_layer
    launches_per_step = 1 if (world == 1 and launches_per_layer == 1) else n_layers * launches_per_layer
    traffic, traffic_src = None, None
    try:   # DRAM bytes / algorithmic bytes from the committed ncu --set full capture of this kernel
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if world == 1 and args.config == "c4":
            traffic = int(tj["ratio"] * bytes_launch)
            traffic_src = "%s (ratio %.3f of algorithmic bytes, scaled to this launch)" % (tj["capture"], tj["ratio"])
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": kname,
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "bytes_per_launch": int(bytes_launch), "launch_us": round(launch_s * 1e6, 2),
                "step_frac": round(float(bytes_step.sum(axis=1).mean()) / (ms_per_step / 1e3) / 1e9 / peak, 4)}

    # ---- e2e through the public C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        xh = xs.cpu().pin_memory()
        yh = torch.empty(B, d).pin_memory()
        barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            i = args.warmup + k
            st = stacks[i % copies]
            if world == 1:
                st.stack.run_host(xh[i], yh)
            else:
                xd = xh[i].to(dev, non_blocking=True)
                st.step(xd, y, None, bufs)
                yh.copy_(y, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": B * args.steps / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": B * d * 4,
               "d2h_bytes_per_step": B * d * 4, "api": "pi_stack_run_host" if world == 1 else
               "host copy + pi_layer_forward + NCCL all_reduce per layer + host copy"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(cfg, args.seed, n_layers, B, args.ref_seconds, dev)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
               "config": workload_config(cfg, B, n_layers, world, {
                   "realised_activity": round(realised, 4),
                   "l2": ("weights rotated over %d layer copies (> L2)" % copies) if single else
                         "inputs larger than L2 (every step streams %d layers; %.1f GB of FFN weights)" % (
                             n_layers, sum(L.info.weight_bytes for L in stacks[0].layers) / 1e9),
                   "algorithmic_MB_per_step": round(float(bytes_step.sum(axis=1).mean()) / 1e6, 2)}, hot_freq=args.hot_freq),
               "latency_ms": {"p50": float(np.percentile(per_step, 50)), "p95": float(np.percentile(per_step, 95)),
                              "p99": float(np.percentile(per_step, 99))},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(args.steps * launches_per_step), "clocks": clk}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- sparse-FFN decode tokens/s and % of the HBM roofline on activated-neuron bytes.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl pi|reference]

With --gpus N > 1 and no torchrun environment (WORLD_SIZE unset), bench.py re-launches itself
under ``torch.distributed.run --nproc-per-node N`` (127.0.0.1 rendezvous), one rank per GPU.
``--dry-run`` exercises the multi-rank plumbing (spawn, rendezvous, the per-layer collective,
max-over-ranks timing, the JSON line) on CPU with gloo and no kernels: its numbers mean nothing.

One step = one decode token (batch B) through every layer of the workload: the whole hot
path of SURVEY.md 8(a) (predictor -> mask -> compaction -> row-sparse up -> column-sparse
down [-> NCCL all-reduce for N > 1]).  Default workload: configs[3] of BASELINE.json, the
Falcon-40B-ReLU FFN stack (d 8192, m 32768, 60 layers, predictor rank 512), the config the
metric's "1/2/4/8 B200" refers to; it fits one GPU (64 GB of FFN weights), so at N = 1 it is
the single-GPU workload and at N > 1 it is neuron-sharded across ranks (strong scaling).
``--config c1`` / ``c2`` (single layers) run the grouped launch (pi_group_run): the SMs split into
independent groups, each decoding its own token through its own chain of layer copies (distinct
seeded weights, so every step streams far more than L2); value = layer-tokens per second.

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
    ap.add_argument("--copies", type=int, default=16, help="layer copies rotated for single-layer configs (--no-group)")
    ap.add_argument("--group-ctas", type=int, default=0,
                    help="single-layer configs: CTAs per independent problem of the grouped launch (pi_group_run); "
                         "0 = the config default (c1: 2, c2: 8)")
    ap.add_argument("--group-layers", type=int, default=4, help="layer copies chained per group (grouped launch)")
    ap.add_argument("--group-defer", type=int, default=0, choices=[0, 1, 2],
                    help="grouped launch: 1/2 = PI_GROUP_DEFER_AFTER_REDUCTION/_BARRIER (pi_group_create flags)")
    ap.add_argument("--no-group", action="store_true",
                    help="single-layer configs: one pi_layer_forward per step over rotated copies instead of the "
                         "grouped launch")
    ap.add_argument("--impl", default="pi", choices=["pi", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=15.0, help="CPU budget of the oracle baseline")
    ap.add_argument("--hot-freq", type=float, default=0.99,
                    help="hot neurons (Insight-1): the fused kernel L2-prefetches the rows of up to --hot-cap "
                         "neurons per layer whose profiled activation frequency is >= this, while the layer "
                         "synchronises after phase 2 (<= 0 disables; c4: 2.22 vs 2.30 ms/step)")
    ap.add_argument("--hot-cap", type=int, default=512, help="hot neurons prefetched per layer (pi_layer_desc.hot_cap)")
    ap.add_argument("--spec-freq", type=float, default=0.0,
                    help="speculative hot prefix (pi_layer_desc.spec_freq): neurons with profiled frequency >= this "
                         "are computed while the grid synchronises after the predictor (<= 0: off, the default -- "
                         "measured slower on c4, DESIGN.md)")
    ap.add_argument("--spec-cap", type=int, default=1 << 30, help="speculative neurons per layer (pi_layer_desc.spec_cap)")
    ap.add_argument("--mean-act", type=float, default=0.10, help="mean activity of the planted profile (5-20%%)")
    ap.add_argument("--rank", dest="pred_rank", type=int, default=None, help="predictor rank r override")
    ap.add_argument("--no-phases", action="store_true", help="skip the traced per-phase breakdown pass")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo plumbing check, no kernels (numbers meaningless)")
    ap.add_argument("--q4", action="store_true", help="INT4 weight-only FFN rows (PI_FFN_Q4, row f3)")
    ap.add_argument("--placement", default="fixed", choices=["fixed", "ilp"],
                    help="per-layer hot-neuron counts: fixed --hot-cap, or the paper's ILP (pi_place_ilp, row f4) "
                         "under --l2-budget-mb")
    ap.add_argument("--l2-budget-mb", type=float, default=60.0, help="fast-tier (L2) budget for --placement ilp")
    return ap.parse_args()


def maybe_spawn(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run, one rank per GPU."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def host_cores():
    """Host core counts the CPU legs can use (cpu_count, affinity, BLAS threads)."""
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = max((p.get("num_threads", 0) for p in threadpool_info()), default=None)
    except Exception:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": aff, "blas_threads": blas, "torch_threads": torch.get_num_threads()}


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
def _oracle_layer_step(O, W, x, cfg, t):
    xo = O.rms_normalize(x) if cfg.rmsnorm else x
    mask, _ = O.predict(xo, W["p_w1"], W["p_b1"], W["p_w2"], W["p_b2"], t)
    ids = O.compact(mask)
    O.sparse_ffn(xo, ids, mask, W["w_up"], W["b_up"], W["w_gate"], W["w_down"], W["b_down"], cfg.act)


def _oracle_time(O, Ws, cfg, B, seed, seconds, max_samples=64):
    """Mean seconds per (token-batch, layer) over a bounded sample (time-boxed, >= 2 samples/layer)."""
    ts = []
    for l, W in enumerate(Ws):
        tok = 0
        while True:
            from paper_2312_12456_b200 import gen
            x = gen.tokens(B, cfg.d, seed=seed + 99, step=tok, device="cpu").numpy().astype(np.float64)
            t0 = time.perf_counter()
            _oracle_layer_step(O, W, x, cfg, W["t"])
            ts.append(time.perf_counter() - t0)
            tok += 1
            if (tok >= 2 and sum(ts) > seconds * (l + 1) / len(Ws)) or tok >= max_samples:
                break
    return float(np.mean(ts)), len(ts)


def _threads(n):
    """Cap NumPy's BLAS and torch's intra-op threads at n (threadpoolctl when present)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n)
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def oracle_baseline(cfg, seed, n_layers_total, B, seconds, device, dims=None):
    """Time oracle predict -> compact -> sparse_ffn on host cores for a bounded sample: once with
    one thread and once with every core of this process's affinity set."""
    from oracle import ffn as O
    from paper_2312_12456_b200 import gen

    k = 2 if n_layers_total > 1 else 1
    t_start = time.perf_counter()
    Ws = []
    for l in range(k):
        w = gen.make_layer(cfg, layer=l, seed=seed, device=device, **(dims or {}))
        f = lambda t: None if t is None else t.float().cpu().numpy()  # noqa: E731
        W = {kk: f(v) for kk, v in w.tensors().items()}
        W["t"] = w.threshold
        Ws.append(W)
        del w
    cores = host_cores()
    with _threads(1):
        per1, n1 = _oracle_time(O, Ws, cfg, B, seed, seconds / 2)
    with _threads(cores["affinity"]):
        perN, nN = _oracle_time(O, Ws, cfg, B, seed, seconds / 2)
    best_cores, per = (1, per1) if per1 <= perN else (cores["affinity"], perN)
    return {"value": B / (per * n_layers_total), "unit": "tokens/s", "cores": best_cores, "kind": "oracle",
            "sample": f"{n1} + {nN} (token-batch, layer) pairs over layers 0..{k - 1} of {n_layers_total}, B={B}, "
                      f"timed with 1 thread and with {cores['affinity']} threads; value = the faster, full-stack "
                      f"time extrapolated x{n_layers_total}; numpy fp64; weight generation and host copies untimed",
            "one_thread_tokens_s": B / (per1 * n_layers_total),
            "all_cores_tokens_s": B / (perN * n_layers_total),
            "ms_per_layer_one_thread": per1 * 1e3, "ms_per_layer_all_cores": perN * 1e3,
            "host": cores, "seconds": round(time.perf_counter() - t_start, 1)}


def run_reference(args, cfg, B, n_layers):
    """--impl reference: the oracle as it stands on the host cores, same config/metric/unit.  One
    step here = one token-batch through ONE layer (a bounded sample of the workload);
    ms_per_step is that measured time, and the metric value extrapolates it x n_layers."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ffn as O
    from paper_2312_12456_b200 import gen

    k = min(2, n_layers)
    Ws = []
    for l in range(k):
        w = gen.make_layer(cfg, layer=l, seed=args.seed, device="cpu", **layer_dims(args))
        f = lambda t: None if t is None else t.float().numpy()  # noqa: E731
        W = {kk: f(v) for kk, v in w.tensors().items()}
        W["t"] = w.threshold
        Ws.append(W)
        del w
    cores = host_cores()

    def one(step):
        W = Ws[step % k]
        x = gen.tokens(B, cfg.d, seed=args.seed, step=step, device="cpu").numpy().astype(np.float64)
        t0 = time.perf_counter()
        _oracle_layer_step(O, W, x, cfg, W["t"])
        return time.perf_counter() - t0

    with _threads(cores["affinity"]):
        for i in range(args.warmup):
            one(i)
        ts = [one(args.warmup + i) for i in range(args.steps)]
    per_layer = float(np.mean(ts))
    value = B / (per_layer * n_layers)
    sample = (f"each step = one token-batch (B={B}) through one of layers 0..{k - 1} (measured); tokens/s = "
              f"B / (mean step time x {n_layers} layers) (extrapolated); numpy fp64, {cores['affinity']} threads")
    out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": per_layer * 1e3, "step": "one token-batch through one layer",
           "ms_per_token_extrapolated": per_layer * n_layers * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference", "config": workload_config(cfg, B, n_layers, args.gpus, args=args),
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores["affinity"], "kind": "oracle",
                            "sample": sample, "host": cores},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def layer_dims(args):
    return {"r": args.pred_rank} if args.pred_rank else {}


def workload_config(cfg, B, n_layers, N, extra=None, args=None):
    hot_freq = args.hot_freq if args is not None else 0.0
    c = {"workload": f"{cfg.name}: {cfg.desc}", "d": cfg.d, "ffn": cfg.m,
         "predictor_rank": (args.pred_rank if args is not None and args.pred_rank else cfg.r),
         "layers": n_layers, "batch": B, "act": cfg.act, "weights": cfg.dtype, "activations": "fp32",
         "mean_activity_target": args.mean_act if args is not None else 0.10,
         "mask_mode": "P (predictor-generated, planted b2)",
         "parallelism": "single GPU" if N == 1 else f"neuron-sharded x{N} (pi_partition) + NCCL all-reduce",
         "hot_neurons": ("L2 prefetch of <= %d neurons/layer with profiled frequency >= %g" %
                         (args.hot_cap, hot_freq)) if hot_freq > 0 else "off",
         "speculative_prefix": ("neurons with profiled frequency >= %g computed while the grid synchronises "
                                "after the predictor, corrected for tokens whose bit is 0" % args.spec_freq)
         if args is not None and args.spec_freq > 0 else "off"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------------------
def phase_breakdown(st, x, y, B, n_layers):
    """One traced (untimed) stack launch: mean over CTAs of each phase of layer 1 (pi_layer_set_trace
    stamps, include/pi.h), in microseconds.  Barriers are the waits after each phase."""
    L0 = st.layers[0]
    P = L0.info.num_sms
    buf = torch.zeros(P * 256, dtype=torch.int64, device=x.device)
    L0.set_trace(buf)
    st.step(x, y, None)
    torch.cuda.synchronize()
    L0.set_trace(None)
    t = buf.view(P, 256)[:, :9].cpu().numpy().astype(np.float64)
    if (t[:, 0] == 0).any() or (t[:, 8] == 0).any():
        return None
    rel = (t - t[:, :1]) / 1e3
    m = rel.mean(axis=0)
    names = ["P1 (a1)", "grid barrier 1", "P2 + threshold (a2)", "grid barrier 2", "compaction (a3)",
             "FFN up+down (a4+a5)", "grid barrier 3", "reduction of partials"]
    out = {nm: round(float(m[i + 1] - m[i]), 2) for i, nm in enumerate(names)}
    out["layer_total"] = round(float(m[8]), 2)
    out["layer_total_max_cta"] = round(float(rel[:, 8].max()), 2)
    out["source"] = "pi_layer_set_trace stamps of layer 1 of one untimed stack launch, mean over CTAs"
    return out


def dry_run(args, cfg, B, n_layers):
    """Multi-rank plumbing on CPU (gloo): spawn/rendezvous, the per-layer all-reduce of [B, d]
    partials, max-over-ranks timing, the JSON line.  No kernels run; the numbers mean nothing."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    d = cfg.d
    x = torch.randn(B, d)
    bufs = [torch.empty(B, d) for _ in range(2)]

    def step():
        cur = x
        for l in range(n_layers):
            dst = bufs[l & 1]
            dst.copy_(cur)
            if world > 1:
                dist.all_reduce(dst)
            cur = dst

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    if world > 1:
        dist.barrier()
    total = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([total])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    if rank == 0:
        out = {"metric": METRIC, "value": B * args.steps / total, "unit": "tokens/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
               "data": "synthetic", "dry_run": True,
               "config": workload_config(cfg, B, n_layers, world, {"note": "CPU gloo plumbing check, no kernels"},
                                         args=args)}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


GROUP_CTAS_DEFAULT = {"c1": 2, "c2": 8}


def run_grouped(args, cfg, B, dev):
    """Single-layer configs (c1, c2): NG independent problems of group_ctas CTAs each in ONE
    persistent launch (pi_group_run); group k chains --group-layers distinct copies of the layer.
    One step = one launch = every group's token through its layer copies."""
    from paper_2312_12456_b200 import gen, pi
    from paper_2312_12456_b200.stack import algorithmic_bytes, build_stack

    pg = args.group_ctas or GROUP_CTAS_DEFAULT.get(cfg.name, 8)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    ng, gl = n_sm // pg, args.group_layers
    stacks = []
    for k in range(ng):
        # no hot-neuron L2 prefetch: every group would pull its own hot rows into the shared L2
        st, _ = build_stack(cfg, n_layers=gl, seed=args.seed + 1000 * k, device=dev, max_batch=1,
                            mean_act=args.mean_act, dims=layer_dims(args))
        if st.stack is not None:
            st.stack.close()          # the group owns the launch
            st.stack = None
        stacks.append(st)
    G = pi.GroupHandle([st.layers for st in stacks], pg, flags=args.group_defer)
    d = cfg.d
    T = args.warmup + args.steps
    xs = torch.stack([torch.cat([gen.tokens(1, d, seed=args.seed + 7 + 31 * k, step=i, device=dev)[None]
                                 for k in range(ng)]) for i in range(T)])          # [T, NG, 1, d]
    y = torch.empty(ng, 1, d, device=dev)
    nbuf = torch.zeros(T, ng, gl, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        G.run(xs[i], y, nbuf[i])
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index or 0)
    clocks.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for k in range(args.steps):
        G.run(xs[args.warmup + k], y, nbuf[args.warmup + k])
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    per_step = np.array([evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)])
    total_ms = evs[0].elapsed_time(evs[-1])
    ms_per_step = total_ms / args.steps
    lt = ng * gl * B                                         # layer-tokens per step
    value = lt * args.steps / (total_ms / 1e3)
    n_host = nbuf.cpu().numpy()[args.warmup:]
    meta = stacks[0].metas[0]
    bytes_step = np.array([sum(algorithmic_bytes(meta, int(v), B) for v in n_host[k].ravel())
                           for k in range(args.steps)])
    realised = float(n_host.mean() / meta.m_local)
    peak, peak_src = hbm_peak()
    l2_bytes = float(torch.cuda.get_device_properties(dev).L2_cache_size)
    launch_s = per_step / 1e3
    achieved = float(bytes_step.mean()) / float(launch_s.mean()) / 1e9
    roofline = {"bound": "hbm", "kernel": "k_layer grouped launch (pi_group_run): %d groups x %d CTAs, %d layer "
                "copies per group" % (ng, pg, gl), "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "traffic_source": None, "peak_source": peak_src,
                "bytes_per_launch": int(bytes_step.mean()), "launch_us": round(float(launch_s.mean()) * 1e6, 2),
                "timing": "CUDA events around each launch inside the timed loop",
                "step_frac": round(float(bytes_step.mean()) / (ms_per_step / 1e3) / 1e9 / peak, 4)}
    e2e = None
    if not args.no_e2e:
        xh = xs.cpu().pin_memory()
        yh = torch.empty(ng, 1, d).pin_memory()
        xd = torch.empty(ng, 1, d, device=dev)
        t0 = time.perf_counter()
        for k in range(args.steps):
            xd.copy_(xh[args.warmup + k], non_blocking=True)
            G.run(xd, y)
            yh.copy_(y, non_blocking=True)
            stream.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e = {"value": lt * args.steps / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": ng * B * d * 4,
               "d2h_bytes_per_step": ng * B * d * 4,
               "api": "pinned host copy + pi_group_run + host copy (GroupHandle.run)"}
    args.hot_freq = 0.0      # reported in config: off for grouped launches
    cpu = None if args.no_cpu_baseline else oracle_baseline(cfg, args.seed, 1, B, args.ref_seconds, dev,
                                                             layer_dims(args))
    out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
           "config": workload_config(cfg, B, 1, 1, {
               "realised_activity": round(realised, 4),
               "grouped": {"groups": ng, "ctas_per_group": pg, "layer_copies_per_group": gl,
                           "flags": args.group_defer,
                           "layer_tokens_per_step": lt,
                           "note": "value = layer-tokens/s: each group decodes its own token through its own "
                                   "chain of distinct layer copies; all groups in one persistent launch"},
               "l2": "%d distinct layer copies, %.0f MB of algorithmic bytes per step (%s the %.0f MB L2)" % (
                   ng * gl, float(bytes_step.mean()) / 1e6,
                   "above" if bytes_step.mean() > l2_bytes else "NOT above", l2_bytes / 1e6),
               "algorithmic_MB_per_step": round(float(bytes_step.mean()) / 1e6, 2)}, args=args),
           "latency_ms": {"p50": float(np.percentile(per_step, 50)), "p95": float(np.percentile(per_step, 95)),
                          "p99": float(np.percentile(per_step, 99))},
           "roofline": roofline, "phases_us": None, "cpu_baseline": cpu, "e2e": e2e,
           "gpu_launches": int(args.steps), "clocks": clk}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    maybe_spawn(args)
    from paper_2312_12456_b200 import gen

    cfg = gen.CONFIGS[args.config]
    B = args.batch or cfg.batch
    n_layers = args.layers or cfg.layers
    if args.impl == "reference":
        run_reference(args, cfg, B, n_layers)
        return
    if args.dry_run:
        dry_run(args, cfg, B, n_layers)
        return

    import torch.distributed as dist
    from paper_2312_12456_b200.stack import algorithmic_bytes, build_stack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1 and n_layers == 1 and not args.no_group and B == 1:
        torch.cuda.set_device(0)
        run_grouped(args, cfg, B, torch.device("cuda", 0))
        return
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    # ---- per-layer hot-neuron counts from the paper's placement ILP (row f4) ----
    ilp_caps, ilp_info = None, None
    if args.placement == "ilp" and args.hot_freq > 0:
        from paper_2312_12456_b200 import pi as _pi
        prof = np.stack([gen.activity_profile(cfg.m, args.mean_act, seed=args.seed, layer=l) for l in range(n_layers)])
        nbytes = [2 * (3 if cfg.act == "reglu" else 2) * cfg.d] * n_layers
        peak_gbs = hbm_peak()[0]
        # fast unit: L2-resident rows (~3x HBM bandwidth), slow: HBM; T_sync: one extra prefetch round
        fast, cnt, obj = _pi.pi_place_ilp(prof, nbytes, 64, args.l2_budget_mb * 1e6, 3 * peak_gbs * 1e9,
                                          peak_gbs * 1e9, 0.5e-6)
        ilp_caps = [int(c) if c > 0 else 1 for c in cnt]
        ilp_info = {"l2_budget_mb": args.l2_budget_mb, "hot_neurons_per_layer": [int(c) for c in cnt],
                    "objective_expected_active_on_fast": round(obj, 2)}
        args.hot_freq = 1e-9   # every neuron is eligible; the ILP count caps each layer

    # ---- build the workload (weights random-init with the config's architecture) ----
    single = n_layers == 1
    copies = args.copies if single else 1
    stacks = []
    for c in range(copies):
        st, _ = build_stack(cfg, n_layers=n_layers, rank=rank, world=world, seed=args.seed + 1000 * c,
                            device=dev, max_batch=B, group=group, mean_act=args.mean_act, dims=layer_dims(args),
                            hot_freq=args.hot_freq if args.hot_freq > 0 else None, hot_cap=args.hot_cap, q4=args.q4,
                            hot_caps=ilp_caps, spec_freq=args.spec_freq, spec_cap=args.spec_cap)
        stacks.append(st)
    d = cfg.d
    T = args.warmup + args.steps
    xs = torch.stack([gen.tokens(B, d, seed=args.seed + 7, step=i, device=dev) for i in range(T)])
    y = torch.empty(B, d, device=dev)
    nbuf = torch.zeros(T, n_layers, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    graphs = None
    if world > 1:
        # the sharded step (per layer: fused kernel + NCCL all-reduce) replays as one CUDA graph
        xg = torch.empty(B, d, device=dev)
        ng = torch.zeros(n_layers, dtype=torch.int32, device=dev)
        graphs = [st.capture(xg, y, ng) for st in stacks]

    def step(i):
        st = stacks[i % copies]
        if graphs is None:
            st.step(xs[i], y, nbuf[i])
        else:
            xg.copy_(xs[i])
            graphs[i % copies].replay()
            nbuf[i].copy_(ng)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up, then EXACTLY K timed steps (one event per step boundary on the launching stream) ----
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
    launches_per_layer = int(stacks[0].layers[0].info.launches_per_forward)
    one_launch = world == 1 and launches_per_layer == 1 and not single
    if world == 1 and launches_per_layer == 1:
        # world 1: every timed step IS one launch of the fused kernel (pi_stack_run: all layers; single-layer
        # configs: one layer), so the per-step events of the timed loop are per-launch durations
        kt = per_step / 1e3
        kb = bytes_step.sum(axis=1)
        timing_src = "CUDA events around each launch inside the timed loop"
    else:
        kt, kb, ar = [], [], []
        for k in range(min(args.steps, 10)):
            i = args.warmup + k
            st = stacks[i % copies]
            e0 = [torch.cuda.Event(enable_timing=True) for _ in range(n_layers)]
            e1 = [torch.cuda.Event(enable_timing=True) for _ in range(n_layers)]
            e2 = [torch.cuda.Event(enable_timing=True) for _ in range(n_layers)]
            cur = xs[i]
            bufs = st._bufs(cur)
            for l, L in enumerate(st.layers):
                dst = bufs[l & 1]
                e0[l].record(stream)
                L.forward(cur, dst)
                e1[l].record(stream)
                if world > 1:
                    dist.all_reduce(dst)
                e2[l].record(stream)
                cur = dst
            torch.cuda.synchronize()
            for l in range(n_layers):
                kt.append(e0[l].elapsed_time(e1[l]) / 1e3)
                ar.append(e1[l].elapsed_time(e2[l]) / 1e3)
                kb.append(algorithmic_bytes(metas[l], int(n_host[k, l]), B))
        timing_src = "CUDA events around each layer's launch in a separate 10-step pass"
    launch_s = float(np.mean(kt))
    bytes_launch = float(np.mean(kb))
    per_rank = None
    if world > 1:
        # the per-GPU view: each rank's fused-layer time, its all-reduce time per
        # layer and the share of the layer's active neurons it owns (the E9 analogue)
        try:
            mine = {"rank": rank, "layer_kernel_us": round(launch_s * 1e6, 2),
                    "allreduce_us_per_layer": round(float(np.mean(ar)) * 1e6, 2),
                    "local_active": round(float(n_host.mean()), 1),
                    "local_activity": round(float(n_host.mean() / metas[0].m_local), 4),
                    "roofline_frac": round(bytes_launch / launch_s / 1e9 / hbm_peak()[0], 4)}
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            tot = sum(r["local_active"] for r in allr)
            for r in allr:
                r["active_share"] = round(r["local_active"] / tot, 4) if tot else None
            per_rank = allr
        except Exception as e:   # diagnostic only: never costs the bench line
            per_rank = {"error": repr(e)}
    peak, peak_src = hbm_peak()
    achieved = bytes_launch / launch_s / 1e9
    kname = ("k_layer x%d layers in one persistent launch (pi_stack_run)" % n_layers) if one_launch else \
        "pi_layer_forward (%d launch(es) per layer)" % launches_per_layer
    launches_per_step = 1 if (world == 1 and launches_per_layer == 1) else n_layers * launches_per_layer
    traffic, traffic_src = None, None
    try:   # DRAM bytes / algorithmic bytes from the committed ncu --set full capture of this kernel
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if one_launch and args.config == tj.get("config", "c4") and B == tj.get("batch", 1):
            traffic = int(tj["ratio"] * bytes_launch)
            traffic_src = "%s (ratio %.3f of algorithmic bytes, scaled to this launch)" % (tj["capture"], tj["ratio"])
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": kname,
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "bytes_per_launch": int(bytes_launch), "launch_us": round(launch_s * 1e6, 2), "timing": timing_src,
                "step_frac": round(float(bytes_step.sum(axis=1).mean()) / (ms_per_step / 1e3) / 1e9 / peak, 4)}

    phases = None
    if world == 1 and one_launch and not args.no_phases:
        try:
            phases = phase_breakdown(stacks[0], xs[0], y, B, n_layers)
        except Exception as e:  # tracing is diagnostic only
            phases = {"error": repr(e)}

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
                xg.copy_(xh[i], non_blocking=True)
                graphs[i % copies].replay()
                yh.copy_(y, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": B * args.steps / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": B * d * 4,
               "d2h_bytes_per_step": B * d * 4, "api": "pi_stack_run_host" if world == 1 else
               "host copy + CUDA-graph replay of (pi_layer_forward + NCCL all_reduce) x layers + host copy"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(cfg, args.seed, n_layers, B, args.ref_seconds, dev, layer_dims(args))

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "int4" if args.q4 else cfg.dtype,
               "data": "synthetic",
               "config": workload_config(cfg, B, n_layers, world, {
                   "realised_activity": round(realised, 4),
                   "l2": ("weights rotated over %d layer copies (> L2)" % copies) if single else
                         "inputs larger than L2 (every step streams %d layers; %.1f GB of FFN weights)" % (
                             n_layers, sum(L.info.weight_bytes for L in stacks[0].layers) / 1e9),
                   "algorithmic_MB_per_step": round(float(bytes_step.sum(axis=1).mean()) / 1e6, 2),
                   "ffn_weights": "INT4 neuron rows (groups of 32, fp16 scales)" if args.q4 else cfg.dtype,
                   "placement": ilp_info or "fixed"}, args=args),
               "latency_ms": {"p50": float(np.percentile(per_step, 50)), "p95": float(np.percentile(per_step, 95)),
                              "p99": float(np.percentile(per_step, 99))},
               "roofline": roofline, "phases_us": phases, "per_rank": per_rank, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(args.steps * launches_per_step), "clocks": clk}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Phase timeline of the fused layer kernel (pi_layer_set_trace): per phase boundary, the
mean and max over CTAs of (stamp - launch start), in microseconds.

  python scripts/trace_layer.py [--config c4] [--reps 20] [--batch 1]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_12456_b200 import gen, pi  # noqa: E402
from paper_2312_12456_b200.stack import algorithmic_bytes, build_stack  # noqa: E402

NAMES = ["start", "P1 done", "grid bar 1", "P2 done", "grid bar 2", "ids ready", "FFN done", "grid bar 3", "end"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--stack", action="store_true", help="trace layer 1 of a pi_stack_run launch")
    ap.add_argument("--hot-freq", type=float, default=0.0, help="hot-neuron L2 prefetch threshold (0 = off)")
    ap.add_argument("--spec-freq", type=float, default=0.0, help="speculative hot prefix threshold (0 = off)")
    ap.add_argument("--q4", action="store_true", help="INT4 FFN rows")
    a = ap.parse_args()
    cfg = gen.CONFIGS[a.config]
    st, _ = build_stack(cfg, n_layers=min(a.layers, cfg.layers), device="cuda", max_batch=a.batch,
                        hot_freq=a.hot_freq if a.hot_freq > 0 else None, spec_freq=a.spec_freq, q4=a.q4)
    P = st.layers[0].info.num_sms
    buf = torch.zeros(P * 256, dtype=torch.int64, device="cuda")
    x = gen.tokens(a.batch, cfg.d, seed=3, device="cuda")
    y = torch.empty_like(x)
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    rows = []
    stage_rows = []
    for rep in range(a.reps):
        L = st.layers[rep % len(st.layers)]
        if a.stack:
            L = st.layers[0]
        L.set_trace(buf)
        buf.zero_()
        if a.stack:
            nn = torch.zeros(len(st.layers), dtype=torch.int32, device="cuda")
            st.stack.run(x, y, nn)
        else:
            L.forward(x, y, None, None, n)
        torch.cuda.synchronize()
        L.set_trace(None)
        if a.stack:
            n = nn[1:2]
        full = buf.view(P, 256).cpu().numpy().astype(np.float64)
        t = full[:, :9]
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        rows.append(rel)
        ready = np.where(full[:, 16:72] > 0, (full[:, 16:72] - t0) / 1e3, np.nan)
        issue = np.where(full[:, 72:128] > 0, (full[:, 72:128] - t0) / 1e3, np.nan)
        stage_rows.append((ready, issue))
        gl = full[:, 200]
        p2d = full[:, 128:192].copy()
        bars = [full[:, 204 + 4 * k:208 + 4 * k].copy() for k in range(4)]
        raw = full[:, 128:192].reshape(P, 16, 4)
        base = raw[:, 0, 3:4]
        dbg = np.where(raw > 0, raw - base[:, :, None] if False else raw - raw[:, :1, 3:4], np.nan)
        x = y.clone()
    R = np.stack(rows[2:])                    # drop warm-up reps
    mean = R.mean(axis=(0, 1))
    mx = R.max(axis=1).mean(axis=0)
    nb = algorithmic_bytes(st.metas[0], int(n.item()), a.batch)
    out = {"config": a.config, "batch": a.batch, "P": P, "bytes_per_layer": nb,
           "phases_us_mean_over_ctas": dict(zip(NAMES, np.round(mean, 2).tolist())),
           "phases_us_max_over_ctas": dict(zip(NAMES, np.round(mx, 2).tolist())),
           "ideal_us_at_peak": round(nb / 6560.6e9 * 1e6, 2)}
    out["g_load_cycles_median_max"] = [float(np.median(gl)), float(gl.max())]
    for k, nm in enumerate(["B1", "B3", "B2", "B4"]):
        bk = bars[k]
        rel_done = (bk[:, 3] - t0) / 1e3
        out[nm + "_cycles_atomret_flagseen_median"] = [float(np.median(bk[:, 1])), float(np.median(bk[:, 2]))]
        out[nm + "_release_us_min_max"] = [float(rel_done.min()), float(rel_done.max())]
    # phase-2 detail (fused.cuh p2_phase, last rep): us relative to the phase-2 entry, median over CTAs
    d0 = p2d[:, 0:1]
    rel = lambda a: np.where(a > 0, (a - d0) / 1e3, np.nan)  # noqa: E731
    out["p2_detail_us_median_over_ctas"] = {
        "g staged": float(np.nanmedian(rel(p2d[:, 1:2]))), "B fragments built": float(np.nanmedian(rel(p2d[:, 2:3]))),
        "first job start (min/max warp)": [float(np.nanmedian(np.nanmin(rel(p2d[:, 16:32]), axis=1))),
                                          float(np.nanmedian(np.nanmax(rel(p2d[:, 16:32]), axis=1)))],
        "first job end (min/max warp)": [float(np.nanmedian(np.nanmin(rel(p2d[:, 48:64]), axis=1))),
                                        float(np.nanmedian(np.nanmax(rel(p2d[:, 48:64]), axis=1)))],
        "mma loop cycles (median/max warp)": [float(np.nanmedian(np.where(p2d[:, 32:48] > 0, p2d[:, 32:48], np.nan))),
                                             float(np.nanmedian(np.nanmax(np.where(p2d[:, 32:48] > 0, p2d[:, 32:48], np.nan), axis=1)))],
        "all logits in zbuf": float(np.nanmedian(rel(p2d[:, 3:4]))),
        "P2 done (ballots)": float(np.nanmedian((full[:, 3] - p2d[:, 0]) / 1e3))}
    rd, iss = stage_rows[-1]
    for cta in (0, P // 2):
        k = int(np.sum(~np.isnan(rd[cta])))
        out[f"cta{cta}_stage_issue_us"] = np.round(iss[cta][:k], 2).tolist()
        out[f"cta{cta}_stage_ready_us"] = np.round(rd[cta][:k], 2).tolist()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-GPU compute of the neuron-sharded step measured on one GPU: rank 0's shard of
every layer (pi_partition, G shards) run as one persistent stack launch, without the per-layer
all-reduce (this sandbox has one GPU).  Prints ms per token, algorithmic bytes and roofline
fraction of the shard -- the compute side of the 1/2/4/8-GPU scaling; the NCCL all-reduce of
B x d fp32 per layer comes on top at G > 1.

    python scripts/shard_compute.py [c4:1,2,4,8 c5:8]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_12456_b200 import gen, pi                      # noqa: E402
from paper_2312_12456_b200.stack import algorithmic_bytes, build_stack   # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
specs = sys.argv[1:] or ["c4:1,2,4,8", "c5:8"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for spec in specs:
    name, gs = spec.split(":")
    cfg = gen.CONFIGS[name]
    for G in [int(g) for g in gs.split(",")]:
        st, _ = build_stack(cfg, n_layers=cfg.layers, rank=0, world=G, seed=0, device=dev, max_batch=1,
                            hot_freq=0.99, hot_cap=512)
        S = pi.StackHandle(st.layers)
        L = len(st.layers)
        steps, warm = 20, 5
        xs = [gen.tokens(1, cfg.d, seed=9, step=i, device=dev) for i in range(steps + warm)]
        y = torch.empty(1, cfg.d, device=dev)
        n = torch.zeros(steps + warm, L, dtype=torch.int32, device=dev)
        for i in range(warm):
            S.run(xs[i], y, n[i])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(warm, warm + steps):
            S.run(xs[i], y, n[i])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        nh = n.cpu().numpy()[warm:]
        by = float(np.mean([sum(algorithmic_bytes(st.metas[l], int(nh[k, l]), 1) for l in range(L))
                            for k in range(steps)]))
        print(json.dumps({"config": name, "G": G, "rank": 0, "layers": L, "m_local": st.metas[0].m_local,
                          "ms_per_token": round(ms, 4), "algorithmic_MB_per_token": round(by / 1e6, 1),
                          "roofline_frac": round(by / (ms / 1e3) / 1e9 / PEAK, 4),
                          "local_activity": round(float(nh.mean() / st.metas[0].m_local), 4),
                          "note": "rank-0 shard only, one persistent launch, no all-reduce (1-GPU sandbox)"}),
              flush=True)
        S.close()
        st.close()
        torch.cuda.empty_cache()

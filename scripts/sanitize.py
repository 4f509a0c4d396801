#!/usr/bin/env python
"""Small, fast workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of libpi on tiny shapes -- the fused persistent kernel (single layer and a
stack, with the hot-neuron prefetch and the speculative prefix), the per-step kernels (B <= 8),
the INT4 per-step kernels and the batched tensor-core path (B = 16).  Prints one line per case.

  compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_12456_b200 import gen, pi  # noqa: E402
from paper_2312_12456_b200.stack import build_stack  # noqa: E402


def main():
    torch.cuda.set_device(0)
    cfg = gen.CONFIGS["c4"]
    dims = {"d": 512, "m": 1024, "r": 32}
    # fused single layer (B = 1, 2) and the per-step path (B = 3)
    w = gen.make_layer(cfg, seed=1, device="cuda", **dims)
    L = pi.Layer(w, max_batch=8)
    for B in (1, 2, 3):
        x = gen.tokens(B, 512, seed=B, device="cuda")
        y = torch.empty_like(x)
        mask, ids = L.new_mask(B), L.new_ids()
        n = torch.zeros(1, dtype=torch.int32, device="cuda")
        L.forward(x, y, mask, ids, n)
        torch.cuda.synchronize()
        print(f"layer B={B}: n_active={int(n.item())} launches={L.info.launches_per_forward if B <= 2 else 'steps'}")
    # stack with hot prefetch + speculative prefix (B = 1)
    st, _ = build_stack(cfg, n_layers=2, seed=2, device="cuda", max_batch=1, dims=dims, hot_freq=0.9,
                        spec_freq=0.99)
    x = gen.tokens(1, 512, seed=5, device="cuda")
    y = torch.empty_like(x)
    st.step(x, y)
    torch.cuda.synchronize()
    print(f"stack L=2 spec={st.layers[0].info.n_spec}: ok")
    st.close()
    # INT4 rows (per-step kernels)
    q = gen.make_q4(w)
    Lq = pi.Layer(w, max_batch=4, q4=q)
    x = gen.tokens(2, 512, seed=6, device="cuda")
    y = torch.empty_like(x)
    Lq.forward(x, y)
    torch.cuda.synchronize()
    print("int4 B=2: ok")
    # batched tensor-core path
    wb = gen.make_layer(gen.CONFIGS["c3"], seed=3, device="cuda", d=512, m=700, r=32)
    Lb = pi.Layer(wb, max_batch=16)
    x = gen.tokens(16, 512, seed=7, device="cuda")
    y = torch.empty_like(x)
    Lb.forward(x, y)
    torch.cuda.synchronize()
    print("batched B=16 (tcgen05): ok", float(np.abs(y.cpu().numpy()).mean()))


if __name__ == "__main__":
    main()

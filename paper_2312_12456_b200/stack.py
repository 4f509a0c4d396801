"""Multi-layer, optionally neuron-sharded decode stacks over libpi handles.

The paper keeps hot neurons on the GPU and cold ones on the CPU, computing
each unit's predicted-active neurons independently and merging the partial
outputs with an add on the GPU.  Here the units are G
identical B200s: ``pi_partition`` places each layer's neurons (equal counts,
balanced expected activity), every rank owns one shard of every layer, and the
merge is one NCCL all-reduce(sum) of the fp32 [B, d] partials per layer over
NVLink.  b_down lives on rank 0 only, so it is added once.

Everything numeric runs in libpi's kernels; this module only builds handles and
sequences calls (plus the NCCL collective).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import gen
from . import pi


@dataclasses.dataclass
class LayerMeta:
    """What the bench needs to count algorithmic bytes for one layer shard."""
    d: int
    m_local: int
    r: int
    reglu: bool
    b_up: bool
    b_down: bool          # this shard owns b_down
    p_b1: bool
    p_b2: bool
    e: int = 2            # bytes per weight element (predictor, biases; 16-bit FFN rows)
    ffn_row_bytes: int = 0  # bytes of one neuron's row per FFN matrix (0: e * d; INT4: codes + scales)


class Stack:
    def __init__(self, layers: List[pi.Layer], metas: List[LayerMeta], rank: int = 0, world: int = 1,
                 group=None):
        self.layers = layers
        self.metas = metas
        self.rank = rank
        self.world = world
        self.group = group
        self.handles = pi.handles(layers)
        self.d = layers[0].d
        # world 1: one persistent launch per step for all layers (pi_stack_run)
        self.stack = pi.StackHandle(layers) if world == 1 else None

    def __len__(self):
        return len(self.layers)

    def step(self, x: torch.Tensor, y: torch.Tensor, n_out: Optional[torch.Tensor] = None,
             bufs: Optional[List[torch.Tensor]] = None, record: Optional[list] = None):
        """One decode step for B tokens through every layer.  World size 1: one pi_stack_run
        call (one persistent launch).  World size > 1: per layer pi_layer_forward on the local
        shard (partial output, b_down on rank 0 only), then all-reduce(sum) of the partials
        (the paper's merge).  ``record`` (tests): each layer's merged output is
        appended to it (world > 1)."""
        if self.world == 1:
            self.stack.run(x, y, n_out)
            return y
        if bufs is None:
            bufs = self._bufs(x)
        cur = x
        for l, L in enumerate(self.layers):
            dst = y if l == len(self.layers) - 1 else bufs[l & 1]
            L.forward(cur, dst, None, None, None if n_out is None else n_out[l:l + 1])
            dist.all_reduce(dst, op=dist.ReduceOp.SUM, group=self.group)
            if record is not None:
                record.append(dst.clone())
            cur = dst
        return y

    def _bufs(self, x: torch.Tensor) -> List[torch.Tensor]:
        key = (x.shape[0], x.device)
        if getattr(self, "_buf_key", None) != key:
            self._buf = [torch.empty(x.shape[0], self.d, device=x.device) for _ in range(2)]
            self._buf_key = key
        return self._buf

    def capture(self, x: torch.Tensor, y: torch.Tensor, n_out: Optional[torch.Tensor] = None):
        """Capture one decode step (static x -> y; every layer's kernel and, for world > 1, its
        NCCL all-reduce) into a CUDA graph; returns the graph -- replay() runs the step with one
        launch from the host.  The caller writes each token into x before replaying."""
        bufs = self._bufs(x)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):           # warm-up on a side stream (NCCL communicator init)
            self.step(x, y, n_out, bufs)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(x, y, n_out, bufs)
        return g

    def close(self):
        if self.stack is not None:
            self.stack.close()
            self.stack = None
        for L in self.layers:
            L.close()


def shard_ids(p: np.ndarray, world: int, rank: int, granule: int = 64) -> Optional[np.ndarray]:
    if world == 1:
        return None
    m = len(p)
    g = granule if m % (granule * world) == 0 else 1
    owner, sids, off = pi.pi_partition(p.astype(np.float32), world, g)
    return sids[off[rank]:off[rank + 1]].copy()


def build_stack(cfg: gen.Config, n_layers: Optional[int] = None, rank: int = 0, world: int = 1, seed: int = 0,
                device="cuda", max_batch: int = 1, mean_act: float = 0.10, group=None,
                keep_weights: bool = False, dims: Optional[dict] = None, hot_freq: Optional[float] = None,
                hot_cap: int = 0, q4: bool = False, hot_caps: Optional[List[int]] = None,
                spec_freq: float = 0.0, spec_cap: int = 1 << 30):
    """Generate the config's layers (random init, seeded) and create this rank's handles.

    Returns (Stack, weights-or-None).  With keep_weights the generator tensors stay alive
    (tests and the oracle baseline read them); otherwise each layer's global tensors are freed
    once the library has its own repacked copy."""
    L = n_layers or cfg.layers
    flags = pi.PI_FLAG_INPUT_RMSNORM if cfg.rmsnorm else 0
    layers, metas, kept = [], [], []
    dims = dims or {}
    for l in range(L):
        w = gen.make_layer(cfg, layer=l, seed=seed, device=device, mean_act=mean_act, **dims)
        nid = shard_ids(w.p, world, rank)
        own = rank == 0
        # the planted activity profile plays the paper's profiler frequencies f_i (Eq. 1)
        freq = None if (hot_freq is None and spec_freq <= 0) else w.p
        qw = gen.make_q4(w) if q4 else None
        layers.append(pi.Layer(w, neuron_ids=nid, max_batch=max_batch, flags=flags, layer_id=l, own_b_down=own,
                               neuron_freq=freq, hot_freq=hot_freq if hot_freq is not None else 2.0,
                               hot_cap=hot_caps[l] if hot_caps is not None else hot_cap, q4=qw,
                               spec_freq=spec_freq, spec_cap=spec_cap))
        del qw
        m_local = w.m if nid is None else len(nid)
        rowb = ((w.d // 2 + w.d // 16 + 15) // 16) * 16 if q4 else 2 * w.d
        metas.append(LayerMeta(w.d, m_local, w.r, w.act == "reglu", w.b_up is not None,
                               own and w.b_down is not None, w.p_b1 is not None, w.p_b2 is not None,
                               ffn_row_bytes=rowb))
        if keep_weights:
            kept.append((w, nid))
        else:
            del w
    if not keep_weights:
        torch.cuda.empty_cache()
    return Stack(layers, metas, rank, world, group), (kept if keep_weights else None)


def algorithmic_bytes(meta: LayerMeta, n_union: int, B: int) -> int:
    """Algorithmic HBM bytes of one layer-step on one shard; counted from the
    realised union count.  Split-K partials, re-reads and over-fetch are NOT algorithmic."""
    e, d, r, m = meta.e, meta.d, meta.r, meta.m_local
    c = 3 if meta.reglu else 2
    row = meta.ffn_row_bytes or e * d
    w = e * (r * d + r * m + (r if meta.p_b1 else 0) + (m if meta.p_b2 else 0))
    w += c * n_union * row + (e * n_union if meta.b_up else 0) + (e * d if meta.b_down else 0)
    words = (m + 31) // 32
    io = 4 * B * d + 4 * B * d + 4 * B * words + 2 * 4 * n_union + 4 * B * r
    return int(w + io)


def algorithmic_flops(meta: LayerMeta, n_union: int, B: int) -> int:
    c = 3 if meta.reglu else 2
    return int(2 * B * (meta.r * meta.d + meta.r * meta.m_local + (c - 1) * n_union * meta.d + n_union * meta.d))

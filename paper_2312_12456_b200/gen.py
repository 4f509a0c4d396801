"""Seeded synthetic workload generator (shared by tests, smoke and bench).

This module holds NONE of the method's arithmetic: no predictor forward, no
FFN, no masking, no compaction.  It only draws random tensors with the shapes
and statistics of the paper's workloads (recipe in DESIGN.md "Input recipe"):

* the activity profile p_i: rank-Zipf p_k = min(1, c k^-s) with c solved for
  the mean activity and s solved so that 80% of activation mass sits in 26% of
  the neurons (OPT-30B), scattered over the index space by a seeded
  permutation (hot neurons 3, 5, 7 are scattered in fig:example);
* layer weights in the ABI's global layouts (include/pi.h), rounded to fp16 or
  bf16 (the paper's FP16 weights);
* the predictor output bias b2, planted from closed-form moments of the
  predictor's hidden layer under x ~ N(0, I) so that P(z_i > 0) ~= p_i
  (a Gaussian moment calculation on the weights, not a forward pass);
* tokens x ~ N(0, I) in fp32 (activations are FP32);
* Bernoulli(p) masks for kernel-isolation runs (SURVEY.md 8(d) mode T) and the
  bit packing of the ABI's mask words;
* integer-exact layers whose every product and partial sum is exact in fp32.

Randomness: torch.Generator seeded from (seed, layer, tensor tag); the same
call on the same device returns the same tensors.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import torch

# --------------------------------------------------------------------------
# configurations (BASELINE.json "configs"; SURVEY.md 8 shapes, reading R14 ranks)
# --------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    d: int
    m: int
    r: int
    act: str            # "relu" | "reglu"
    bias: bool          # OPT-style biases present
    layers: int
    dtype: str          # "f16" | "bf16"
    rmsnorm: bool       # PI_FLAG_INPUT_RMSNORM for chained stacks (reading R19)
    batch: int = 1
    desc: str = ""


CONFIGS = {
    "c1": Config("c1", 768, 3072, 64, "relu", True, 1, "f16", False, 1,
                 "single OPT-125M-shaped FFN layer d=768 ffn=3072, batch 1, predictor rank 64"),
    "c2": Config("c2", 4096, 16384, 256, "relu", True, 1, "f16", False, 1,
                 "OPT-6.7B FFN layer d=4096 ffn=16384, batch 1, predictor rank 256, 1 GPU"),
    "c3": Config("c3", 5120, 13824, 320, "reglu", False, 40, "bf16", True, 1,
                 "ReLU-Llama-13B gated FFN d=5120 ffn=13824, 40-layer stack, batch 1-8"),
    "c4": Config("c4", 8192, 32768, 512, "relu", False, 60, "bf16", True, 1,
                 "Falcon-40B-ReLU FFN d=8192 ffn=32768, 60 layers, neuron-sharded"),
    "c5": Config("c5", 12288, 49152, 768, "relu", True, 96, "f16", True, 1,
                 "OPT-175B FFN d=12288 ffn=49152, 96 layers, neuron-sharded across 8 GPUs"),
}

TORCH_DTYPE = {"f16": torch.float16, "bf16": torch.bfloat16}

_TAGS = {"w_up": 1, "w_gate": 2, "w_down": 3, "b_up": 4, "b_down": 5,
         "p_w1": 6, "p_w2": 7, "p_b1": 8, "x": 9, "mask": 10, "perm": 11}


def _gen(seed: int, layer: int, tag: str, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(layer) * 1_009 + _TAGS[tag] * 7_919) & ((1 << 62) - 1))
    return g


# --------------------------------------------------------------------------
# activity profile (power law; reading R12)
# --------------------------------------------------------------------------


def _zipf_probs(m: int, mean_act: float, s: float) -> np.ndarray:
    k = np.arange(1, m + 1, dtype=np.float64)
    base = k ** (-s)
    lo, hi = 0.0, 1.0 / base[-1]
    for _ in range(200):              # bisection on c: mean(min(1, c k^-s)) = mean_act
        c = 0.5 * (lo + hi)
        if np.minimum(1.0, c * base).mean() < mean_act:
            lo = c
        else:
            hi = c
    return np.minimum(1.0, 0.5 * (lo + hi) * base)


def mass_fraction(p: np.ndarray, mass: float = 0.8) -> float:
    """Smallest fraction of neurons carrying ``mass`` of the total activation mass."""
    q = np.sort(np.asarray(p, dtype=np.float64))[::-1]
    c = np.cumsum(q) / q.sum()
    return float(np.searchsorted(c, mass) + 1) / len(q)


def solve_zipf_s(m: int, mean_act: float, top_frac: float = 0.26, mass: float = 0.8) -> float:
    """s such that ``mass`` of the activations come from ``top_frac`` of the neurons."""
    lo, hi = 0.05, 6.0
    for _ in range(60):
        s = 0.5 * (lo + hi)
        if mass_fraction(_zipf_probs(m, mean_act, s), mass) > top_frac:
            lo = s                    # too flat: steepen
        else:
            hi = s
    return 0.5 * (lo + hi)


def activity_profile(m: int, mean_act: float = 0.10, seed: int = 0, layer: int = 0,
                     s: Optional[float] = None) -> np.ndarray:
    """p_i in index order: rank-Zipf probabilities scattered by a seeded permutation."""
    if s is None:
        s = solve_zipf_s(m, mean_act)
    p_rank = _zipf_probs(m, mean_act, s)
    perm = torch.randperm(m, generator=_gen(seed, layer, "perm", "cpu")).numpy()
    p = np.empty(m, dtype=np.float64)
    p[perm] = p_rank
    return p


# --------------------------------------------------------------------------
# layer weights
# --------------------------------------------------------------------------


@dataclasses.dataclass
class LayerWeights:
    """One FFN layer in the ABI's GLOBAL layouts (include/pi.h pi_layer_desc)."""
    d: int
    m: int
    r: int
    act: str
    w_up: torch.Tensor                 # [m, d]
    w_gate: Optional[torch.Tensor]     # [m, d] (reglu)
    w_down: torch.Tensor               # [d, m]  nn.Linear fc2.weight
    b_up: Optional[torch.Tensor]       # [m]
    b_down: Optional[torch.Tensor]     # [d]
    p_w1: torch.Tensor                 # [r, d]
    p_b1: Optional[torch.Tensor]       # [r]
    p_w2: torch.Tensor                 # [m, r]
    p_b2: Optional[torch.Tensor]       # [m]
    threshold: float = 0.0
    pred_act: str = "relu"
    p: Optional[np.ndarray] = None     # target activity profile used for b2

    def tensors(self):
        return {k: getattr(self, k) for k in ("w_up", "w_gate", "w_down", "b_up", "b_down",
                                              "p_w1", "p_b1", "p_w2", "p_b2")}


def _randn(shape, std, gen, device, dtype):
    t = torch.randn(*shape, generator=gen, device=device, dtype=torch.float32)
    t.mul_(std)
    return t.to(dtype)


def _ndtri(q: np.ndarray) -> np.ndarray:
    """Inverse standard normal CDF (Acklam's rational approximation, |err| < 1.2e-9)."""
    a = [-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
         1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00]
    b = [-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
         6.680131188771972e+01, -1.328068155288572e+01]
    c = [-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
         -2.549671010115381e+00, 4.374664141464968e+00, 2.938163982698783e+00]
    dd = [7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
          3.754408661907416e+00]
    q = np.clip(np.asarray(q, dtype=np.float64), 1e-15, 1 - 1e-15)
    out = np.empty_like(q)
    lo = q < 0.02425
    hi = q > 1 - 0.02425
    mid = ~(lo | hi)
    t = np.sqrt(-2 * np.log(q[lo]))
    out[lo] = (((((c[0] * t + c[1]) * t + c[2]) * t + c[3]) * t + c[4]) * t + c[5]) / \
        ((((dd[0] * t + dd[1]) * t + dd[2]) * t + dd[3]) * t + 1)
    t = np.sqrt(-2 * np.log(1 - q[hi]))
    out[hi] = -(((((c[0] * t + c[1]) * t + c[2]) * t + c[3]) * t + c[4]) * t + c[5]) / \
        ((((dd[0] * t + dd[1]) * t + dd[2]) * t + dd[3]) * t + 1)
    qm = q[mid] - 0.5
    t = qm * qm
    out[mid] = (((((a[0] * t + a[1]) * t + a[2]) * t + a[3]) * t + a[4]) * t + a[5]) * qm / \
        (((((b[0] * t + b[1]) * t + b[2]) * t + b[3]) * t + b[4]) * t + 1)
    return out


def plant_b2(p_w1: torch.Tensor, p_w2: torch.Tensor, p: np.ndarray, pred_act: str = "relu",
             threshold: float = 0.0, x_var: float = 1.0) -> torch.Tensor:
    """Choose b2 so that P(z_i > t) ~= p_i for x ~ N(0, x_var I).

    Closed-form moments: u_j ~ N(0, s_j^2) with s_j^2 = x_var ||P1_j||^2.  For the ReLU
    hidden layer E[relu(u)] = s/sqrt(2 pi), Var = s^2 (1/2 - 1/(2 pi)); z^0_i = P2_i . g is
    approximately N(mu_i, sig_i^2) with mu_i = sum_j P2_ij E[g_j], sig_i^2 = sum_j P2_ij^2 Var(g_j).
    b2_i = t - mu_i - sig_i Phi^-1(1 - p_i);  p_i = 1 -> 10 sigma margin.
    Returned in p_w2's dtype and device.
    """
    w1 = p_w1.double().cpu()
    w2 = p_w2.double().cpu()
    s2 = x_var * (w1 * w1).sum(dim=1)
    if pred_act == "relu":
        mean_g = torch.sqrt(s2) / math.sqrt(2 * math.pi)
        var_g = s2 * (0.5 - 1.0 / (2 * math.pi))
    else:
        mean_g = torch.zeros_like(s2)
        var_g = s2
    mu = (w2 * mean_g[None, :]).sum(dim=1).numpy()
    sig = np.sqrt((w2 * w2 * var_g[None, :]).sum(dim=1).numpy())
    pc = np.clip(p, 0.0, 1.0)
    zq = np.where(pc >= 1.0, -10.0, np.where(pc <= 0.0, 10.0, _ndtri(1.0 - np.clip(pc, 1e-12, 1 - 1e-12))))
    b2 = threshold - mu - sig * zq
    return torch.from_numpy(b2).to(device=p_w2.device, dtype=p_w2.dtype)


def make_layer(cfg: Config, layer: int = 0, seed: int = 0, device="cpu", dtype: Optional[str] = None,
               mean_act: float = 0.10, pred_act: str = "relu", threshold: float = 0.0,
               m: Optional[int] = None, d: Optional[int] = None, r: Optional[int] = None) -> LayerWeights:
    """Random-init layer with the config's architecture (no trained weights exist)."""
    d = d or cfg.d
    m = m or cfg.m
    r = r or cfg.r
    td = TORCH_DTYPE[dtype or cfg.dtype]
    dev = torch.device(device)
    w_up = _randn((m, d), 1.0 / math.sqrt(d), _gen(seed, layer, "w_up", dev), dev, td)
    w_gate = _randn((m, d), 1.0 / math.sqrt(d), _gen(seed, layer, "w_gate", dev), dev, td) \
        if cfg.act == "reglu" else None
    w_down = _randn((d, m), math.sqrt(2.0 / (mean_act * m)), _gen(seed, layer, "w_down", dev), dev, td)
    b_up = _randn((m,), 0.02, _gen(seed, layer, "b_up", dev), dev, td) if cfg.bias else None
    b_down = _randn((d,), 0.02, _gen(seed, layer, "b_down", dev), dev, td) if cfg.bias else None
    p_w1 = _randn((r, d), 1.0 / math.sqrt(d), _gen(seed, layer, "p_w1", dev), dev, td)
    p_w2 = _randn((m, r), 1.0 / math.sqrt(r), _gen(seed, layer, "p_w2", dev), dev, td)
    p = activity_profile(m, mean_act, seed, layer)
    p_b2 = plant_b2(p_w1, p_w2, p, pred_act, threshold)
    return LayerWeights(d, m, r, cfg.act, w_up, w_gate, w_down, b_up, b_down,
                        p_w1, None, p_w2, p_b2, threshold, pred_act, p)


def tokens(B: int, d: int, seed: int = 0, step: int = 0, device="cpu") -> torch.Tensor:
    """x ~ N(0, I), fp32 [B, d]."""
    return torch.randn(B, d, generator=_gen(seed, step, "x", device), device=device, dtype=torch.float32)


# --------------------------------------------------------------------------
# mode-T masks and the ABI bit layout
# --------------------------------------------------------------------------


def bernoulli_masks(p: np.ndarray, B: int, seed: int = 0, step: int = 0) -> torch.Tensor:
    """Independent Bernoulli(p_i) masks, bool [B, m] (SURVEY 8(d) mode T)."""
    u = torch.rand(B, len(p), generator=_gen(seed, step, "mask", "cpu"), dtype=torch.float64)
    return u < torch.from_numpy(np.asarray(p, dtype=np.float64))[None, :]


def pack_bits(mask: torch.Tensor) -> torch.Tensor:
    """bool [B, m] -> int32 view of uint32 words [B, ceil(m/32)]; bit (i & 31) of word i >> 5."""
    mask = mask.reshape(mask.shape[0], -1).to(torch.int64).cpu()
    B, m = mask.shape
    nw = (m + 31) // 32
    pad = torch.zeros(B, nw * 32, dtype=torch.int64)
    pad[:, :m] = mask
    shifts = torch.arange(32, dtype=torch.int64)
    words = (pad.view(B, nw, 32) << shifts).sum(dim=2)
    return torch.from_numpy(words.numpy().astype(np.uint32).view(np.int32).copy())


# --------------------------------------------------------------------------
# integer-exact layers (bitwise pins)
# --------------------------------------------------------------------------


def make_int_layer(d: int, m: int, r: int, act: str = "relu", seed: int = 0, bias: bool = True,
                   dtype: str = "bf16", device="cpu") -> LayerWeights:
    """Small-integer weights: every product and partial sum is exact in fp32 in any order.

    ReLU: weights in {-2..2}, x in {-3..3}, d <= 256, m <= 1024.  ReGLU: weights in
    {-1, 0, 1}, x in {-2..2}, d <= 64, m <= 256.  Predictor: P1, P2 in {-1, 0, 1},
    r <= 64, integer b2, threshold 0.5 (integer logits never tie).
    """
    if act == "relu":
        assert d <= 256 and m <= 1024
        lo, hi = -2, 2
    else:
        assert d <= 64 and m <= 256
        lo, hi = -1, 1
    assert r <= 64
    g = torch.Generator().manual_seed(seed)
    td = TORCH_DTYPE[dtype]

    def ri(shape, a, b):
        return torch.randint(a, b + 1, shape, generator=g).to(td).to(device)

    w_up = ri((m, d), lo, hi)
    w_gate = ri((m, d), lo, hi) if act == "reglu" else None
    w_down = ri((d, m), lo, hi)
    b_up = ri((m,), -3, 3) if bias else None
    b_down = ri((d,), -3, 3) if bias else None
    p_w1 = ri((r, d), -1, 1)
    p_b1 = ri((r,), -2, 2) if bias else None
    p_w2 = ri((m, r), -1, 1)
    # negative integer offsets give ~10-40% activity; bound checks: |z| <= r * d * 3 + |b2|
    p_b2 = torch.randint(-int(2 * math.sqrt(d * r)), 1, (m,), generator=g).to(td).to(device)
    return LayerWeights(d, m, r, act, w_up, w_gate, w_down, b_up, b_down,
                        p_w1, p_b1, p_w2, p_b2, 0.5, "relu", None)


def int_tokens(B: int, d: int, act: str = "relu", seed: int = 0, device="cpu") -> torch.Tensor:
    g = torch.Generator().manual_seed(seed + 12345)
    a = 3 if act == "relu" else 2
    return torch.randint(-a, a + 1, (B, d), generator=g).to(torch.float32).to(device)


# ---------------------------------------------------------------------------
# INT4 neuron rows (row f3; format: DESIGN.md reading R21, oracle/quant.py): model preparation,
# i.e. input generation -- the method's arithmetic (dequantise + FFN) runs in libpi / the oracle.
# ---------------------------------------------------------------------------
Q4_GROUP = 32


def quantize_q4(w: torch.Tensor):
    """Symmetric 4-bit quantisation of rows [rows, d] (d % 32 == 0) in groups of 32: scale =
    fp16(max|w| / 7), code = clamp(round(w / scale), -8, 7) + 8, two codes per byte (element 2k in
    the low nibble of byte k).  Returns (codes uint8 [rows, d/2], scales fp16 [rows, d/32])."""
    rows, d = w.shape
    assert d % Q4_GROUP == 0
    wf = w.float().reshape(rows, d // Q4_GROUP, Q4_GROUP)
    amax = wf.abs().amax(dim=2)
    scale = (amax / 7.0).to(torch.float16)
    s = scale.float()
    q = torch.where(s[..., None] > 0, torch.round(wf / torch.where(s > 0, s, 1.0)[..., None]), torch.zeros_like(wf))
    q = (q.clamp(-8, 7) + 8).to(torch.uint8).reshape(rows, d)
    codes = (q[:, 0::2] | (q[:, 1::2] << 4)).contiguous()
    return codes, scale.contiguous()


@dataclasses.dataclass
class Q4Weights:
    """The FFN of one layer as INT4 neuron rows (neuron-major: row i = neuron i's d-vector)."""
    up_codes: torch.Tensor
    up_scales: torch.Tensor
    gate_codes: Optional[torch.Tensor]
    gate_scales: Optional[torch.Tensor]
    down_codes: torch.Tensor            # neuron i's down column W_down[:, i] as a row
    down_scales: torch.Tensor


def make_q4(w: "LayerWeights") -> Q4Weights:
    """Quantise a generated layer's FFN matrices (the predictor keeps its 16-bit weights)."""
    uc, us = quantize_q4(w.w_up)
    gc, gs = quantize_q4(w.w_gate) if w.w_gate is not None else (None, None)
    dc, ds = quantize_q4(w.w_down.t().contiguous())
    return Q4Weights(uc, us, gc, gs, dc, ds)

"""CPU oracle for PowerInfer's predictor-gated sparse FFN (arXiv 2312.12456).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  It shares no code with the CUDA path (``paper_2312_12456_b200/``) and
imports nothing from it.

Everything is plain NumPy in float64.  Weights arrive as arrays holding exact
fp16/bf16 values (e.g. ``tensor.float().numpy()``) and are upcast to float64
here, so the only rounding is the fp64 arithmetic itself.

Citations: ``P:n`` = line n of the paper's text, ``S:n`` = line n of
SPEC.md (used for interfaces and worked examples only).  Step names O0..O7
follow SURVEY.md section 8(c).

Layouts (the ABI's global layouts, include/pi.h):
  x       [B, d]            token activations (fp32 in the ABI)
  w_up    [m, d]            FC1: row i = neuron i                   (P:107 footnote)
  w_gate  [m, d]            ReGLU gate rows (act == "reglu")
  w_down  [d, m]            FC2 (nn.Linear layout): column i = neuron i
  p_w1    [r, d], p_b1 [r]  predictor input->hidden layer
  p_w2    [m, r], p_b2 [m]  predictor hidden->output layer
"""
from __future__ import annotations

import numpy as np

RMS_EPS = 1e-6  # DESIGN.md reading R19 (harness pre-FFN norm); not from the paper


def f64(a):
    """Upcast to float64 (exact for fp16/bf16/fp32 inputs)."""
    return np.asarray(a, dtype=np.float64)


def _rowdot(rows, x):
    """Dot product of every row with every token: out[b, k] = sum_j rows[k, j] * x[b, j].

    Written as an elementwise product followed by a sum along the contiguous
    axis, so the value for row k does not depend on which other rows are
    present (NumPy reduces each row independently).  This is what makes the
    'exact mask equals dense' pin (OI-2) hold bit for bit.
    """
    rows = f64(rows)
    x = f64(x)
    out = np.empty((x.shape[0], rows.shape[0]), dtype=np.float64)
    step = max(1, (1 << 22) // max(1, rows.shape[1]))  # bound the temporary
    for b in range(x.shape[0]):
        for k0 in range(0, rows.shape[0], step):
            out[b, k0:k0 + step] = (rows[k0:k0 + step] * x[b][None, :]).sum(axis=1)
    return out


def rms_normalize(x):
    """O0 (PI_FLAG_INPUT_RMSNORM): x_hat = x / sqrt(mean(x^2) + 1e-6), per token.

    Not from the paper: the harness stand-in for the model's pre-FFN norm when
    FFN layers are chained without attention (reading R19).
    """
    x = f64(x)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + RMS_EPS)


def predict(x, p_w1, p_b1, p_w2, p_b2, threshold, pred_act="relu"):
    """O1: the adaptive predictor, an MLP with one hidden layer.

      u = P1 x + b1 ; g = relu(u) (pred_act="relu") or g = u ("linear")
      z = P2 g + b2 ; neuron i predicted active iff z_i > t          (reading R3)

    t is a logit threshold: t = 0 is SPEC's sigmoid(z) > 0.5.
    NaN logits compare False, i.e. inactive.
    Returns (mask bool [B, m], z float64 [B, m]).
    """
    x = f64(np.atleast_2d(x))
    u = _rowdot(p_w1, x)
    if p_b1 is not None:
        u = u + f64(p_b1)[None, :]
    if pred_act == "relu":
        g = np.maximum(u, 0.0)
    elif pred_act == "linear":
        g = u
    else:
        raise ValueError(pred_act)
    z = _rowdot(p_w2, g)
    if p_b2 is not None:
        z = z + f64(p_b2)[None, :]
    with np.errstate(invalid="ignore"):
        mask = z > float(threshold)
    return mask, z


def compact(mask):
    """O2: ascending ids of neurons active for ANY token of the batch (union; reading R9).

    For B = 1 this is SPEC's canonical ascending, duplicate-free active set.
    """
    mask = np.atleast_2d(np.asarray(mask, dtype=bool))
    return np.flatnonzero(mask.any(axis=0)).astype(np.int32)


def _act_rows(x, ids, w_up, b_up, w_gate, act):
    """Pre-activation a and activated h for the rows ``ids`` (reading R5/R6)."""
    ids = np.asarray(ids, dtype=np.int64)
    a = _rowdot(np.asarray(w_up)[ids], x)
    if b_up is not None:
        a = a + f64(b_up)[ids][None, :]          # bias before the activation
    if act == "relu":
        h = np.maximum(a, 0.0)
    elif act == "reglu":
        gt = _rowdot(np.asarray(w_gate)[ids], x)  # gate carries no bias (reading R6)
        h = np.maximum(gt, 0.0) * a
    else:
        raise ValueError(act)
    return a, h


def _down(h, ids, w_down, b_down, d):
    """O4: y_b = b_down + sum over ids in ascending order of h[b, k] * W_down[:, ids[k]]."""
    B = h.shape[0]
    y = np.zeros((B, d), dtype=np.float64)
    if b_down is not None:
        y += f64(b_down)[None, :]
    wd = np.asarray(w_down)
    for k, i in enumerate(np.asarray(ids, dtype=np.int64)):
        y += h[:, k:k + 1] * f64(wd[:, i])[None, :]
    return y


def sparse_ffn(x, ids, mask, w_up, b_up, w_gate, w_down, b_down, act="relu"):
    """O3 + O4: the neuron-aware FFN restricted to ``ids``.

    For every id i (ascending) and token b:
      a = W_up[i] . x_b + b_up[i]
      h = relu(a)                      (ReLU)
      h = relu(W_gate[i] . x_b) * a    (ReGLU, reading R5)
      h := 0 if token b's own mask bit for i is 0   (per-token semantics, reading R9)
    y_b = b_down + sum_i h_{b,i} W_down[:, i]

    ``mask`` is bool [B, m] (or None: every id counts for every token).
    Pass x already normalised (rms_normalize) when the layer uses the norm flag.
    Returns y float64 [B, d].
    """
    x = f64(np.atleast_2d(x))
    ids = np.asarray(ids, dtype=np.int64)
    d = x.shape[1]
    if ids.size == 0:
        return _down(np.zeros((x.shape[0], 0)), ids, w_down, b_down, d)
    _, h = _act_rows(x, ids, w_up, b_up, w_gate, act)
    if mask is not None:
        keep = np.atleast_2d(np.asarray(mask, dtype=bool))[:, ids]
        h = np.where(keep, h, 0.0)
    return _down(h, ids, w_down, b_down, d)


def sparse_hidden(x, ids, mask, w_up, b_up, w_gate, act="relu"):
    """O3 alone: h [B, n] for the rows ``ids`` with per-token masking (for kernel-level parity)."""
    x = f64(np.atleast_2d(x))
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        return np.zeros((x.shape[0], 0))
    _, h = _act_rows(x, ids, w_up, b_up, w_gate, act)
    if mask is not None:
        keep = np.atleast_2d(np.asarray(mask, dtype=bool))[:, ids]
        h = np.where(keep, h, 0.0)
    return h


def dense_ffn(x, w_up, b_up, w_gate, w_down, b_down, act="relu"):
    """O6: the unmasked FFN y = b_down + W_down act(W_up x + b_up) (P:177-205 fig:bg-mlp).

    Written as two plain matrix products (a library primitive), a different
    route from sparse_ffn's gather + ordered accumulation.
    """
    x = f64(np.atleast_2d(x))
    a = x @ f64(w_up).T
    if b_up is not None:
        a = a + f64(b_up)[None, :]
    if act == "relu":
        h = np.maximum(a, 0.0)
    else:
        h = np.maximum(x @ f64(w_gate).T, 0.0) * a
    y = h @ f64(w_down).T
    if b_down is not None:
        y = y + f64(b_down)[None, :]
    return y


def dense_ffn_ordered(x, w_up, b_up, w_gate, w_down, b_down, act="relu"):
    """O6 in sparse_ffn's summation order: sparse_ffn over all m ids with no mask."""
    m = np.asarray(w_up).shape[0]
    return sparse_ffn(x, np.arange(m), None, w_up, b_up, w_gate, w_down, b_down, act)


def exact_mask(x, w_up, b_up, w_gate, act="relu"):
    """O7: the true activation set (reading R4).

    ReLU: {i : W_up[i] . x + b_up[i] > 0}; ReGLU: {i : W_gate[i] . x > 0}.
    Returns bool [B, m].
    """
    x = f64(np.atleast_2d(x))
    m = np.asarray(w_up).shape[0]
    ids = np.arange(m)
    if act == "relu":
        a, _ = _act_rows(x, ids, w_up, b_up, None, "relu")
        return a > 0.0
    return _rowdot(w_gate, x) > 0.0


def merge(partials):
    """O5: y = sum of the per-unit partial outputs, in unit order."""
    out = None
    for p in partials:
        out = f64(p).copy() if out is None else out + f64(p)
    return out


def pack_mask(mask):
    """Pack bool [B, m] into the ABI's uint32 words [B, ceil(m/32)]: bit (i & 31) of word i >> 5."""
    mask = np.atleast_2d(np.asarray(mask, dtype=bool))
    B, m = mask.shape
    nw = (m + 31) // 32
    words = np.zeros((B, nw), dtype=np.uint64)
    for i in range(m):
        words[:, i >> 5] |= mask[:, i].astype(np.uint64) << np.uint64(i & 31)
    return words.astype(np.uint32)


def unpack_mask(words, m):
    """Inverse of pack_mask."""
    words = np.atleast_2d(np.asarray(words, dtype=np.uint32)).astype(np.uint64)
    i = np.arange(m)
    return ((words[:, i >> 5] >> (i & 31).astype(np.uint64)) & np.uint64(1)).astype(bool)


def near_threshold(z, threshold, band=1e-4):
    """Neurons whose oracle logit is within ``band`` of t: their mask bits are "don't care"
    in parity (BASELINE.json north_star tolerance)."""
    return np.abs(f64(z) - float(threshold)) <= band


def rel_l2(y, ref):
    """||y - ref||_2 / ||ref||_2 (north_star output tolerance metric); inf if ref == 0 and y != 0."""
    y = f64(y)
    ref = f64(ref)
    nr = np.linalg.norm(ref)
    ne = np.linalg.norm(y - ref)
    if nr == 0.0:
        return 0.0 if ne == 0.0 else np.inf
    return ne / nr

"""CPU oracle for INT4 weight-only neuron rows.

TEST INFRASTRUCTURE ONLY (see oracle/ffn.py header): imported only by tests/,
__graft_entry__.smoke() and bench.py's CPU legs; shares no code with the CUDA path.

The paper evaluates "FP16 and INT4 quantized parameters, with intermediate activations in
FP32" and reports INT4 inference ("Inference with Quantization"),
but never states the INT4 format.  PowerInfer is built on llama.cpp, whose basic
4-bit format is symmetric with one scale per block of 32 weights; reading R21 fixes
this build's format:

  * a neuron's d-vector (its up row, gate row, or down column W_down[:, i]) is cut into
    groups of 32 consecutive elements (d % 32 == 0);
  * group g stores a scale s_g (an fp16 value) and 32 codes q in 0..15;
  * the weight is w = s_g * (q - 8)                                   (step O9)
  * codes are packed two per byte, element 2k in the low nibble and element 2k + 1 in the
    high nibble of byte k of the row; a row of d weights is d / 2 bytes of codes and d / 32
    fp16 scales.

After O9 the FFN is the plain one of oracle/ffn.py on the dequantised rows (O3-O4): the method
with INT4 weights is the method with the weights those codes represent.
"""
from __future__ import annotations

import numpy as np

GROUP = 32


def dequantize_rows(codes, scales):
    """O9: w[i, j] = scales[i, j // 32] * (q[i, j] - 8) in float64 (exact: an fp16 scale times a
    small integer).  codes uint8 [rows, d/2] (two codes per byte, low nibble first), scales
    fp16-valued [rows, d/32]."""
    codes = np.asarray(codes, dtype=np.uint8)
    rows, half = codes.shape
    d = 2 * half
    q = np.empty((rows, d), dtype=np.int64)
    q[:, 0::2] = codes & 0x0F
    q[:, 1::2] = codes >> 4
    s = np.asarray(scales, dtype=np.float64)
    assert s.shape == (rows, d // GROUP), (s.shape, rows, d)
    return np.repeat(s, GROUP, axis=1) * (q - 8).astype(np.float64)


def sparse_ffn_q4(x, ids, mask, up_codes, up_scales, b_up, gate_codes, gate_scales, down_codes, down_scales,
                  b_down, act="relu"):
    """O9 then O3-O4: the sparse FFN over INT4 neuron rows.  down_codes/down_scales hold each
    neuron's down vector as a row (neuron-major [m, d/2] / [m, d/32]); the FFN oracle takes
    W_down in the nn.Linear layout [d, m], hence the transpose."""
    from . import ffn as O
    ids = np.asarray(ids, dtype=np.int64)
    # only the rows the step touches are dequantised; the FFN sees them in the same ascending order
    sub = np.arange(len(ids))
    w_up = dequantize_rows(np.asarray(up_codes)[ids], np.asarray(up_scales)[ids])
    w_gate = None if gate_codes is None else dequantize_rows(np.asarray(gate_codes)[ids], np.asarray(gate_scales)[ids])
    w_down = dequantize_rows(np.asarray(down_codes)[ids], np.asarray(down_scales)[ids]).T
    b_sub = None if b_up is None else np.asarray(b_up)[ids]
    m_sub = None if mask is None else np.atleast_2d(np.asarray(mask, dtype=bool))[:, ids]
    return O.sparse_ffn(x, sub, m_sub, w_up, b_sub, w_gate, w_down, b_down, act)

"""Pins the INT4 dequantisation step O9 (oracle/quant.py, reading R21) to things other
than itself: closed-form code values, a pure-Python bit-twiddling twin over every byte value,
nibble order on a ramp, the fp16 scale range, and the paper's worked example (fig:example,
P:489-505) run through INT4 rows (integer weights with scale 1 are exact, so the answers are the
golden y = [6, 23], ReGLU [18, 69])."""
import numpy as np
import pytest

from oracle import ffn as O
from oracle import quant as Q


def _scalar_dequant(codes_row, scales_row):
    """Independent twin: per element, pick the nibble with shifts and masks in pure Python."""
    out = []
    for j in range(2 * len(codes_row)):
        byte = int(codes_row[j // 2])
        q = (byte >> (4 * (j % 2))) & 15
        out.append(float(scales_row[j // 32]) * (q - 8))
    return out


def test_closed_form_codes():
    s = np.float16(0.5)
    codes = np.zeros((1, 16), np.uint8)
    codes[0, 0] = 0x80      # element 0: q = 0 -> -8 s ; element 1: q = 8 -> 0
    codes[0, 1] = 0xF7      # element 2: q = 7 -> -s ; element 3: q = 15 -> 7 s
    codes[0, 2:] = 0x88     # the rest: 0
    w = Q.dequantize_rows(codes, np.array([[s]], np.float16))
    assert w.shape == (1, 32)
    assert w[0, :4].tolist() == [-4.0, 0.0, -0.5, 3.5]
    assert (w[0, 4:] == 0).all()


def test_every_byte_value_against_scalar_twin():
    rng = np.random.default_rng(0)
    codes = np.arange(256, dtype=np.uint8).reshape(8, 32)            # every byte value once
    scales = rng.standard_normal((8, 2)).astype(np.float16)
    w = Q.dequantize_rows(codes, scales)
    for i in range(8):
        assert w[i].tolist() == _scalar_dequant(codes[i], scales[i])


def test_nibble_order_on_a_ramp():
    # q_j = j mod 16 for j < 64: byte k = (2k mod 16) | ((2k + 1) mod 16) << 4
    d = 64
    q = np.arange(d) % 16
    codes = (q[0::2] | (q[1::2] << 4)).astype(np.uint8)[None, :]
    w = Q.dequantize_rows(codes, np.ones((1, 2), np.float16))
    assert w[0].tolist() == (q - 8).astype(float).tolist()


def test_group_scales_apply_to_their_32_elements():
    codes = np.full((1, 48), 0x99, np.uint8)                           # q = 9 everywhere -> +1 * s
    scales = np.array([[1.0, -2.0, 65504.0]], np.float16)              # incl. the largest fp16
    w = Q.dequantize_rows(codes, scales)
    assert (w[0, :32] == 1.0).all() and (w[0, 32:64] == -2.0).all() and (w[0, 64:] == 65504.0).all()


def _golden_q4(golden, act):
    """fig:example weights (integers in [-2, 2]) as INT4 rows with scale 1: codes = w + 8."""
    d = 32

    def rows(a):
        a = np.asarray(a, dtype=np.int64)
        full = np.zeros((a.shape[0], d), np.int64)
        full[:, :a.shape[1]] = a
        q = full + 8
        return (q[:, 0::2] | (q[:, 1::2] << 4)).astype(np.uint8), np.ones((a.shape[0], 1), np.float16)

    gate = rows(golden["w_up"])
    up = rows(golden["cases"]["G6_reglu"]["w_up_reglu"]) if act == "reglu" else gate
    down = rows(golden["w_down_T"])
    return up, gate, down


@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_golden_example_through_int4_rows(golden, act):
    (uc, us), (gc, gs), (dc, ds) = _golden_q4(golden, act)
    x = np.zeros((1, 32))
    x[0, :2] = [1, 2]
    ids = np.array(golden["cases"]["G1_predict"]["ids"])
    mask = np.zeros((1, 8), bool)
    mask[0, ids] = True
    y = Q.sparse_ffn_q4(x, ids, mask, uc, us, None, gc if act == "reglu" else None,
                        gs if act == "reglu" else None, dc, ds, None, act)
    exp = golden["cases"]["G6_reglu"]["y"][0] if act == "reglu" else golden["cases"]["G2_sparse_ffn"]["y"][0]
    assert y[0, :2].tolist() == exp and (y[0, 2:] == 0).all()


def test_q4_ffn_equals_ffn_on_dequantised_rows():
    """sparse_ffn_q4 is O9 composed with the (separately pinned) O3-O4, bit for bit."""
    rng = np.random.default_rng(3)
    m, d, B = 40, 64, 2
    uc = rng.integers(0, 256, (m, d // 2), dtype=np.uint8)
    dc = rng.integers(0, 256, (m, d // 2), dtype=np.uint8)
    us = (rng.random((m, d // 32)) * 0.1).astype(np.float16)
    ds = (rng.random((m, d // 32)) * 0.1).astype(np.float16)
    x = rng.standard_normal((B, d))
    mask = rng.random((B, m)) < 0.3
    ids = O.compact(mask)
    y = Q.sparse_ffn_q4(x, ids, mask, uc, us, None, None, None, dc, ds, None, "relu")
    ref = O.sparse_ffn(x, ids, mask, Q.dequantize_rows(uc, us), None, None, Q.dequantize_rows(dc, ds).T, None, "relu")
    assert (y == ref).all()
    # empty id set: y = b_down
    b = rng.standard_normal(d)
    y0 = Q.sparse_ffn_q4(x, np.array([], np.int64), np.zeros((B, m), bool), uc, us, None, None, None, dc, ds, b,
                         "relu")
    assert (y0 == b[None, :]).all()


def test_generator_quantiser_round_trip():
    """gen.quantize_q4 (input preparation) produces codes whose dequantisation is within half a
    step of the original weights, with each group's largest |w| hitting code 8 +/- 7."""
    import torch
    from paper_2312_12456_b200 import gen
    g = torch.Generator().manual_seed(1)
    w = torch.randn(7, 96, generator=g).to(torch.bfloat16)
    codes, scales = gen.quantize_q4(w)
    assert codes.dtype == torch.uint8 and codes.shape == (7, 48) and scales.shape == (7, 3)
    wq = Q.dequantize_rows(codes.numpy(), scales.float().numpy())
    step = np.repeat(scales.float().numpy(), 32, axis=1)
    err = np.abs(wq - w.float().numpy())
    assert (err <= 0.5 * step * (1 + 1e-3) + 1e-6).all()

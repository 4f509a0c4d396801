"""GPU parity of the INT4 weight-only FFN path (PI_FFN_Q4, row f3) against the oracle's O9 + O3-O4
(oracle/quant.py): golden example and integer layers bit for bit, random layers within the
north_star tolerance (rel-L2 <= 1e-3, internal gate 1e-5) with the oracle fed the GPU's own ids
and mask bits, at several tiles, ragged m, B = 1..8 and one full-size c4 layer."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import ffn as O
from oracle import quant as Q

pytestmark = pytest.mark.gpu

TOL = 1e-3
GATE = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_12456_b200 import gen, pi
    torch.cuda.set_device(0)
    return gen, pi


def f(t):
    return None if t is None else t.float().cpu().numpy()


def _q4_exact(w_int: torch.Tensor):
    """Integer rows [rows, d] in [-8, 7] as INT4 rows with scale 1 (codes = w + 8): exact."""
    q = (w_int.to(torch.int64) + 8).to(torch.uint8).cpu()
    codes = (q[:, 0::2] | (q[:, 1::2] << 4)).contiguous()
    scales = torch.ones(w_int.shape[0], w_int.shape[1] // 32, dtype=torch.float16)
    return codes.cuda(), scales.cuda()


def _q4_of(gen, w, exact=False):
    if not exact:
        return gen.make_q4(w)
    uc, us = _q4_exact(w.w_up.float())
    gc, gs = _q4_exact(w.w_gate.float()) if w.w_gate is not None else (None, None)
    dc, ds = _q4_exact(w.w_down.float().t().contiguous())
    return gen.Q4Weights(uc, us, gc, gs, dc, ds)


def _run(L, x):
    B = x.shape[0]
    y = torch.full((B, L.d), float("nan"), device="cuda")
    mask = L.new_mask(B)
    ids = L.new_ids()
    n = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    L.forward(x, y, mask, ids, n)
    torch.cuda.synchronize()
    nn = int(n.item())
    return y.cpu().numpy(), O.unpack_mask(mask.cpu().numpy().view(np.uint32), L.m_local), ids[:nn].cpu().numpy()


def _oracle(w, q4, x, gm, gids, norm=False):
    xo = f(x).astype(np.float64)
    if norm:
        xo = O.rms_normalize(xo)
    om, z = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), w.threshold, w.pred_act)
    band = O.near_threshold(z, w.threshold)
    assert ((gm == om) | band).all()
    assert (gids == O.compact(gm)).all()
    return Q.sparse_ffn_q4(xo, gids, gm, f(q4.up_codes).astype(np.uint8), f(q4.up_scales), f(w.b_up),
                           None if q4.gate_codes is None else f(q4.gate_codes).astype(np.uint8), f(q4.gate_scales),
                           f(q4.down_codes).astype(np.uint8), f(q4.down_scales), f(w.b_down), w.act)


@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_golden_example_q4(env, act):
    """fig:example with INT4 FFN rows of scale 1: y = [6, 23] (ReLU), [18, 69] (ReGLU)."""
    gen, pi = env
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "fig_example.json")))
    d, m, r = 32, 8, 8

    def pad(a, rows, cols):
        out = torch.zeros(rows, cols)
        a = torch.tensor(a, dtype=torch.float32)
        out[: a.shape[0], : a.shape[1]] = a
        return out

    gate = pad(g["w_up"], m, d)
    up = pad(g["cases"]["G6_reglu"]["w_up_reglu"], m, d) if act == "reglu" else gate
    wdT = pad(g["w_down_T"], m, d)
    cu = lambda t: t.to(torch.bfloat16).cuda().contiguous()  # noqa: E731
    w = gen.LayerWeights(d, m, r, act, cu(up), cu(gate) if act == "reglu" else None, cu(wdT.T.contiguous()), None,
                         None, cu(pad(g["p_w1"], r, d)), None, cu(pad(g["p_w2"], m, r)), None, g["threshold"], "relu",
                         None)
    q4 = _q4_of(gen, w, exact=True)
    L = pi.Layer(w, max_batch=2, q4=q4)
    assert L.info.ffn_format == pi.PI_FFN_Q4
    x = torch.zeros(1, d, device="cuda")
    x[0, :2] = torch.tensor([1.0, 2.0])
    y, gm, ids = _run(L, x)
    assert ids.tolist() == [3, 4, 5]
    exp = g["cases"]["G6_reglu"]["y"][0] if act == "reglu" else g["cases"]["G2_sparse_ffn"]["y"][0]
    assert y[0, :2].tolist() == exp and (y[0, 2:] == 0).all()
    if act == "relu":   # G7: batch of two with per-token masks
        c = g["cases"]["G7_batch2"]
        x2 = torch.zeros(2, d, device="cuda")
        x2[:, :2] = torch.tensor(c["x"], dtype=torch.float32)
        y2, gm2, ids2 = _run(L, x2)
        assert ids2.tolist() == c["union_ids"] and (y2[:, :2] == np.array(c["y"])).all()


@pytest.mark.parametrize("act,shape", [("relu", (256, 1000, 64)), ("reglu", (64, 250, 16))])
@pytest.mark.parametrize("B", [1, 3, 8])
def test_integer_layers_q4_bitwise(env, act, shape, B):
    gen, pi = env
    d, m, r = shape
    w = gen.make_int_layer(d, m, r, act, seed=d + m + B, dtype="bf16", device="cuda")
    q4 = _q4_of(gen, w, exact=True)
    L = pi.Layer(w, max_batch=8, q4=q4)
    x = gen.int_tokens(B, d, act, seed=B).cuda()
    y, gm, ids = _run(L, x)
    yo = _oracle(w, q4, x, gm, ids)
    assert (y == yo).all()


@pytest.mark.parametrize("name,dims", [("c1", (768, 3072, 64)), ("c2", (4096, 2048, 256)),
                                       ("c3", (5120, 1400, 320)), ("c4", (8192, 1000, 512))])
@pytest.mark.parametrize("B", [1, 4, 8])
def test_random_layers_q4(env, name, dims, B):
    gen, pi = env
    cfg = gen.CONFIGS[name]
    d, m, r = dims
    w = gen.make_layer(cfg, seed=7, device="cuda", d=d, m=m, r=r)
    q4 = _q4_of(gen, w)
    flags = pi.PI_FLAG_INPUT_RMSNORM if cfg.rmsnorm else 0
    L = pi.Layer(w, max_batch=8, flags=flags, q4=q4)
    x = gen.tokens(B, d, seed=11, device="cuda") * (3.0 if cfg.rmsnorm else 1.0)
    y, gm, ids = _run(L, x)
    yo = _oracle(w, q4, x, gm, ids, norm=cfg.rmsnorm)
    err = O.rel_l2(y, yo)
    assert err <= TOL and err <= GATE, err


def test_empty_and_full_masks_q4(env):
    gen, pi = env
    cfg = gen.CONFIGS["c1"]
    w = gen.make_layer(cfg, seed=1, device="cuda", d=512, m=700, r=32)
    q4 = _q4_of(gen, w)
    x = gen.tokens(3, 512, device="cuda")
    L = pi.Layer(w, max_batch=4, threshold=float("inf"), q4=q4)
    y, gm, ids = _run(L, x)
    assert len(ids) == 0 and (y == np.tile(f(w.b_down), (3, 1))).all()
    L = pi.Layer(w, max_batch=4, threshold=float("-inf"), q4=q4)
    y, gm, ids = _run(L, x)
    assert len(ids) == 700
    yo = Q.sparse_ffn_q4(f(x), ids, gm, f(q4.up_codes).astype(np.uint8), f(q4.up_scales), f(w.b_up), None, None,
                         f(q4.down_codes).astype(np.uint8), f(q4.down_scales), f(w.b_down), "relu")
    assert O.rel_l2(y, yo) <= GATE


def test_full_size_c4_layer_q4(env):
    gen, pi = env
    cfg = gen.CONFIGS["c4"]
    w = gen.make_layer(cfg, seed=0, device="cuda")
    q4 = _q4_of(gen, w)
    L = pi.Layer(w, max_batch=1, q4=q4)
    assert L.info.weight_bytes < 0.4 * 2 * 2 * cfg.m * cfg.d   # INT4 rows: ~0.28x the 16-bit FFN bytes
    x = gen.tokens(1, cfg.d, seed=1, device="cuda")
    y, gm, ids = _run(L, x)
    yo = _oracle(w, q4, x, gm, ids)
    assert O.rel_l2(y, yo) <= GATE
    assert 0.03 < gm.mean() < 0.3

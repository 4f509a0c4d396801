"""Pins the oracle (oracle/ffn.py) to mathematics that does not depend on it:

* OI-1  all-ones mask == the dense FFN computed by torch.nn.functional.linear in fp64
        (a library routine, different code route), and == the ordered dense path bit for bit;
* OI-2  the exact ReLU/ReGLU mask == dense, bit for bit (skipped terms are exact zeros);
* OI-3  brute force: every mask of a tiny layer vs the scalar loop twin (oracle/scalar.py);
* additivity over disjoint masks; permutation equivariance;
* integer-exact layers vs exact int64 arithmetic (no rounding anywhere);
* predictor boundary cases and the threshold/sigmoid equivalence (reading R3);
* compaction vs brute force sorted(set(...)), popcount == count;
* RMS normalisation closed form.
"""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import ffn as O
from oracle import scalar as S


def _rand_layer(rng, d, m, r, act="relu", bias=True):
    L = dict(
        w_up=rng.standard_normal((m, d)) / np.sqrt(d),
        w_gate=rng.standard_normal((m, d)) / np.sqrt(d) if act == "reglu" else None,
        w_down=rng.standard_normal((d, m)) / np.sqrt(m),
        b_up=rng.standard_normal(m) * 0.1 if bias else None,
        b_down=rng.standard_normal(d) * 0.1 if bias else None,
        p_w1=rng.standard_normal((r, d)) / np.sqrt(d),
        p_b1=rng.standard_normal(r) * 0.1 if bias else None,
        p_w2=rng.standard_normal((m, r)) / np.sqrt(r),
        p_b2=rng.standard_normal(m) * 0.5 - 0.5 if bias else None,
    )
    # round to bf16 values like the real workload (exact in fp64)
    for k, v in L.items():
        if v is not None:
            L[k] = torch.from_numpy(v).to(torch.bfloat16).double().numpy()
    return L


def _torch_dense(x, L, act):
    """Independent dense FFN via torch fp64 library routines."""
    xt = torch.from_numpy(np.asarray(x, dtype=np.float64))
    t = lambda a: None if a is None else torch.from_numpy(a)  # noqa: E731
    a = F.linear(xt, t(L["w_up"]), t(L["b_up"]))
    h = F.relu(a) if act == "relu" else F.relu(F.linear(xt, t(L["w_gate"]))) * a
    return F.linear(h, t(L["w_down"]), t(L["b_down"])).numpy()


@pytest.mark.parametrize("act", ["relu", "reglu"])
@pytest.mark.parametrize("bias", [True, False])
def test_oi1_all_ones_equals_dense(act, bias):
    rng = np.random.default_rng(11)
    d, m, r, B = 48, 96, 16, 3
    L = _rand_layer(rng, d, m, r, act, bias)
    x = rng.standard_normal((B, d))
    ones = np.ones((B, m), dtype=bool)
    y = O.sparse_ffn(x, np.arange(m), ones, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], act)
    ref = _torch_dense(x, L, act)
    assert O.rel_l2(y, ref) < 1e-13
    assert O.rel_l2(O.dense_ffn(x, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], act), ref) < 1e-13
    yo = O.dense_ffn_ordered(x, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], act)
    assert (y == yo).all()


@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_oi2_exact_mask_equals_dense_bitwise(act):
    rng = np.random.default_rng(12)
    d, m, r, B = 40, 120, 8, 4
    L = _rand_layer(rng, d, m, r, act)
    x = rng.standard_normal((B, d))
    em = O.exact_mask(x, L["w_up"], L["b_up"], L["w_gate"], act)
    assert 0 < em.sum() < em.size
    y = O.sparse_ffn(x, O.compact(em), em, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], act)
    yo = O.dense_ffn_ordered(x, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], act)
    assert (y == yo).all()
    assert O.rel_l2(y, _torch_dense(x, L, act)) < 1e-13
    # exact mask really is the support of h
    h = O.sparse_hidden(x, np.arange(m), None, L["w_up"], L["b_up"], L["w_gate"], act)
    assert ((h != 0) == em).all()


@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_oi3_brute_force_all_masks(act):
    """Every one of the 2^m masks of a tiny layer, numpy oracle vs scalar loop twin."""
    rng = np.random.default_rng(13)
    d, m = 5, 10
    L = _rand_layer(rng, d, m, 4, act)
    x = rng.standard_normal(d)
    for bits in range(1 << m):
        active = [(bits >> i) & 1 == 1 for i in range(m)]
        ids = [i for i in range(m) if active[i]]
        y = O.sparse_ffn([x], ids, None, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], act)[0]
        ys = S.ffn_masked(list(x), active, L["w_up"].tolist(), L["b_up"].tolist(),
                          None if L["w_gate"] is None else L["w_gate"].tolist(),
                          L["w_down"].tolist(), L["b_down"].tolist(), act)
        np.testing.assert_allclose(y, ys, rtol=1e-12, atol=1e-12)


def test_predict_vs_scalar_twin():
    rng = np.random.default_rng(14)
    d, m, r = 7, 16, 5
    L = _rand_layer(rng, d, m, r)
    for t in (-0.3, 0.0, 0.4):
        for pa in ("relu", "linear"):
            x = rng.standard_normal(d)
            mask, z = O.predict([x], L["p_w1"], L["p_b1"], L["p_w2"], L["p_b2"], t, pa)
            ref = S.predict(list(x), L["p_w1"].tolist(), L["p_b1"].tolist(), L["p_w2"].tolist(),
                            L["p_b2"].tolist(), t, pa)
            near = O.near_threshold(z, t, 1e-12)[0]
            assert all(mask[0][i] == ref[i] for i in range(m) if not near[i])


def test_additivity_disjoint_masks():
    """y(S u T) - b = (y(S) - b) + (y(T) - b) for disjoint S, T."""
    rng = np.random.default_rng(15)
    d, m = 32, 64
    L = _rand_layer(rng, d, m, 8)
    x = rng.standard_normal((2, d))
    perm = rng.permutation(m)
    Sset, Tset = np.sort(perm[:20]), np.sort(perm[20:45])
    U = np.sort(np.concatenate([Sset, Tset]))
    f = lambda ids, bd: O.sparse_ffn(x, ids, None, L["w_up"], L["b_up"], None, L["w_down"], bd)  # noqa: E731
    yS, yT, yU = f(Sset, None), f(Tset, None), f(U, None)
    assert O.rel_l2(yS + yT, yU) < 1e-14
    assert O.rel_l2(f(U, L["b_down"]) - L["b_down"], yU) < 1e-14


def test_permutation_equivariance():
    rng = np.random.default_rng(16)
    d, m, r = 24, 48, 8
    L = _rand_layer(rng, d, m, r, "reglu")
    x = rng.standard_normal((3, d))
    mask, z = O.predict(x, L["p_w1"], L["p_b1"], L["p_w2"], L["p_b2"], 0.0)
    y = O.sparse_ffn(x, O.compact(mask), mask, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], "reglu")
    P = rng.permutation(m)
    mask2, z2 = O.predict(x, L["p_w1"], L["p_b1"], L["p_w2"][P], L["p_b2"][P], 0.0)
    assert (mask2 == mask[:, P]).all()
    y2 = O.sparse_ffn(x, O.compact(mask2), mask2, L["w_up"][P], L["b_up"][P], L["w_gate"][P],
                      L["w_down"][:, P], L["b_down"], "reglu")
    assert O.rel_l2(y2, y) < 1e-14


@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_integer_layer_exact_vs_int64(act):
    """Integer weights and inputs: the oracle's fp64 result equals exact int64 arithmetic."""
    rng = np.random.default_rng(17)
    d, m, r, B = (64, 200, 16, 3)
    lo = -2 if act == "relu" else -1
    ri = lambda *s: rng.integers(lo, -lo + 1, s).astype(np.int64)  # noqa: E731
    w_up, w_gate, w_down = ri(m, d), ri(m, d), ri(d, m)
    b_up, b_down = rng.integers(-3, 4, m), rng.integers(-3, 4, d)
    p_w1, p_w2 = rng.integers(-1, 2, (r, d)), rng.integers(-1, 2, (m, r))
    p_b2 = rng.integers(-20, 1, m)
    x = rng.integers(-3, 4, (B, d)).astype(np.int64)
    # exact integer reference
    g = np.maximum(x @ p_w1.T, 0)
    z = g @ p_w2.T + p_b2
    mask_ref = z > 0.5
    a = x @ w_up.T + b_up
    h = np.maximum(a, 0) if act == "relu" else np.maximum(x @ w_gate.T, 0) * a
    h = np.where(mask_ref, h, 0)
    y_ref = h @ w_down.T + b_down
    mask, zo = O.predict(x, p_w1, None, p_w2, p_b2, 0.5)
    assert (zo == z).all() and (mask == mask_ref).all()
    y = O.sparse_ffn(x, O.compact(mask), mask, w_up, b_up, w_gate if act == "reglu" else None,
                     w_down, b_down, act)
    assert (y == y_ref).all()


def test_predictor_boundaries():
    """S:219 strongly negative rows -> empty; S:220 threshold 'probability 0' (t = -inf) -> all;
    t = +inf -> none; NaN logits inactive; sigmoid(z) > 0.5 <=> z > 0 (reading R3)."""
    rng = np.random.default_rng(18)
    d, m, r = 16, 40, 8
    L = _rand_layer(rng, d, m, r)
    x = rng.standard_normal((2, d))
    mask, _ = O.predict(x, L["p_w1"], None, L["p_w2"], np.full(m, -1e9), 0.0)
    assert not mask.any()
    mask, _ = O.predict(x, L["p_w1"], None, -np.abs(L["p_w2"]) * 0, np.full(m, -1e9), -np.inf)
    assert mask.all()
    mask, _ = O.predict(x, L["p_w1"], L["p_b1"], L["p_w2"], L["p_b2"], np.inf)
    assert not mask.any()
    b2 = L["p_b2"].copy()
    b2[3] = np.nan
    mask, z = O.predict(x, L["p_w1"], L["p_b1"], L["p_w2"], b2, -np.inf)
    assert not mask[:, 3].any() and mask[:, [0, 1, 2, 4]].all()
    mask, z = O.predict(x, L["p_w1"], L["p_b1"], L["p_w2"], L["p_b2"], 0.0)
    sig = 1.0 / (1.0 + np.exp(-z))
    assert ((sig > 0.5) == mask).all()


def test_compact_brute_force():
    rng = np.random.default_rng(19)
    for B, m in [(1, 1), (1, 31), (1, 32), (3, 33), (8, 300), (2, 1000)]:
        mask = rng.random((B, m)) < 0.2
        ids = O.compact(mask)
        ref = sorted(set(i for b in range(B) for i in range(m) if mask[b, i]))
        assert ids.tolist() == ref
        union = np.zeros(m, bool)
        union[ids] = True
        words = O.pack_mask(union[None])
        assert sum(bin(int(w)).count("1") for w in words[0]) == len(ids)
        assert (O.unpack_mask(O.pack_mask(mask), m) == mask).all()


def test_pack_mask_bit_layout():
    m = 70
    mask = np.zeros((1, m), bool)
    mask[0, [0, 31, 32, 69]] = True
    w = O.pack_mask(mask)[0]
    assert w.tolist() == [1 | (1 << 31), 1, 1 << 5]


def test_rms_normalize_closed_form():
    x = np.array([[3.0, 4.0], [0.0, 0.0]])
    xn = O.rms_normalize(x)
    assert np.allclose(xn[0], np.array([3.0, 4.0]) / np.sqrt(12.5 + 1e-6), rtol=0, atol=1e-15)
    assert (xn[1] == 0).all()
    # relu(s a) = s relu(a): normalising commutes with the ReLU FFN up to the scalar
    rng = np.random.default_rng(20)
    L = _rand_layer(rng, 16, 32, 4, bias=False)
    xx = rng.standard_normal((1, 16)) * 7
    s = 1.0 / np.sqrt(np.mean(xx ** 2) + 1e-6)
    y1 = O.dense_ffn(O.rms_normalize(xx), L["w_up"], None, None, L["w_down"], None)
    y2 = O.dense_ffn(xx, L["w_up"], None, None, L["w_down"], None) * s
    assert O.rel_l2(y1, y2) < 1e-14


def test_rel_l2_definition():
    assert O.rel_l2([3.0, 4.0], [3.0, 4.0]) == 0.0
    assert O.rel_l2([0.0, 0.0], [0.0, 0.0]) == 0.0
    assert O.rel_l2([1e-30, 0.0], [0.0, 0.0]) == np.inf
    assert abs(O.rel_l2([3.0, 5.0], [3.0, 4.0]) - 0.2) < 1e-15


def test_near_threshold_band():
    z = np.array([0.49995, 0.5, 0.50011, 0.7])
    assert O.near_threshold(z, 0.5).tolist() == [True, True, False, False]


@pytest.mark.parametrize("B", [1, 2, 8])
def test_batch_equals_independent_tokens(B):
    rng = np.random.default_rng(21 + B)
    L = _rand_layer(rng, 32, 64, 8, "reglu")
    x = rng.standard_normal((B, 32))
    mask, _ = O.predict(x, L["p_w1"], L["p_b1"], L["p_w2"], L["p_b2"], 0.0)
    y = O.sparse_ffn(x, O.compact(mask), mask, L["w_up"], L["b_up"], L["w_gate"], L["w_down"], L["b_down"], "reglu")
    for b in range(B):
        yb = O.sparse_ffn(x[b:b + 1], O.compact(mask[b:b + 1]), mask[b:b + 1], L["w_up"], L["b_up"],
                          L["w_gate"], L["w_down"], L["b_down"], "reglu")
        assert O.rel_l2(yb[0], y[b]) < 1e-14


def test_itertools_sanity():
    # the brute-force suites above enumerate masks with bit tricks; keep an independent count
    assert sum(1 for _ in itertools.product([0, 1], repeat=10)) == 1 << 10

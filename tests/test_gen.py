"""Checks that the seeded workload generator produces the paper's workload statistics."""
import numpy as np
import torch

from oracle import ffn as O
from paper_2312_12456_b200 import gen


def test_zipf_profile_calibration():
    """mean activity ~10% and 80% of activation mass in 26% of the neurons."""
    for m in (3072, 16384, 32768):
        p = gen.activity_profile(m, 0.10, seed=0)
        assert abs(p.mean() - 0.10) < 1e-6
        assert abs(gen.mass_fraction(p) - 0.26) < 0.01
        assert p.max() == 1.0          # an always-on prefix exists (~3%)
        assert 0.01 < (p >= 1.0).mean() < 0.06
    s = gen.solve_zipf_s(32768, 0.10)
    assert 1.15 < s < 1.35             # s ~= 1.25


def test_profile_is_scattered_and_seeded():
    p0 = gen.activity_profile(4096, 0.1, seed=0)
    p1 = gen.activity_profile(4096, 0.1, seed=0)
    p2 = gen.activity_profile(4096, 0.1, seed=1)
    assert (p0 == p1).all() and not (p0 == p2).all()
    hot = np.flatnonzero(p0 >= 1.0)
    assert hot.min() < 4096 // 4 and hot.max() > 3 * 4096 // 4   # hot neurons are scattered


def test_planted_predictor_activity():
    """Mode P: masks from the planted predictor realise the target per-neuron rates."""
    cfg = gen.CONFIGS["c1"]
    L = gen.make_layer(cfg, seed=3)
    x = gen.tokens(400, cfg.d, seed=3).numpy()
    f = lambda t: None if t is None else t.float().numpy()  # noqa: E731
    mask, _ = O.predict(x, f(L.p_w1), f(L.p_b1), f(L.p_w2), f(L.p_b2), L.threshold)
    act = mask.mean()
    assert 0.08 < act < 0.12
    rate = mask.mean(axis=0)
    assert np.corrcoef(rate, L.p)[0, 1] > 0.9
    per_tok = mask.sum(axis=1) / cfg.m
    assert per_tok.std() > 0.005     # per-token activity varies


def test_layer_shapes_and_dtypes():
    for name in ("c1", "c3"):
        cfg = gen.CONFIGS[name]
        L = gen.make_layer(cfg, m=256, d=128, r=16)
        assert L.w_up.shape == (256, 128) and L.w_down.shape == (128, 256)
        assert L.p_w1.shape == (16, 128) and L.p_w2.shape == (256, 16) and L.p_b2.shape == (256,)
        assert (L.w_gate is not None) == (cfg.act == "reglu")
        assert L.w_up.dtype == gen.TORCH_DTYPE[cfg.dtype]


def test_layer_determinism():
    cfg = gen.CONFIGS["c1"]
    a = gen.make_layer(cfg, layer=2, seed=5, m=128, d=64, r=8)
    b = gen.make_layer(cfg, layer=2, seed=5, m=128, d=64, r=8)
    c = gen.make_layer(cfg, layer=3, seed=5, m=128, d=64, r=8)
    assert torch.equal(a.w_up, b.w_up) and torch.equal(a.p_b2, b.p_b2)
    assert not torch.equal(a.w_up, c.w_up)


def test_pack_bits_matches_oracle_layout():
    rng = np.random.default_rng(0)
    for B, m in [(1, 5), (2, 64), (3, 100), (8, 3072)]:
        mask = torch.from_numpy(rng.random((B, m)) < 0.3)
        w = gen.pack_bits(mask).numpy().view(np.uint32)
        assert (w == O.pack_mask(mask.numpy())).all()


def test_bernoulli_masks_rate():
    p = gen.activity_profile(8192, 0.1, seed=1)
    mk = gen.bernoulli_masks(p, 64, seed=1)
    assert abs(mk.float().mean().item() - 0.1) < 0.01


def test_integer_layers_bounds():
    """The fp32-exactness premise of the integer pins: every partial sum is < 2^24."""
    for act, (d, m, r) in (("relu", (256, 1024, 64)), ("reglu", (64, 256, 64))):
        L = gen.make_int_layer(d, m, r, act, seed=1)
        x = gen.int_tokens(4, d, act).numpy().astype(np.int64)
        I = lambda t: t.float().numpy().astype(np.int64)  # noqa: E731
        a_abs = np.abs(x) @ np.abs(I(L.w_up)).T + np.abs(I(L.b_up))
        if act == "relu":
            h_abs = a_abs
        else:
            h_abs = (np.abs(x) @ np.abs(I(L.w_gate)).T) * a_abs
        y_abs = h_abs @ np.abs(I(L.w_down)).T + np.abs(I(L.b_down))
        assert y_abs.max() < 2 ** 24
        u_abs = np.abs(x) @ np.abs(I(L.p_w1)).T + np.abs(I(L.p_b1))
        z_abs = u_abs @ np.abs(I(L.p_w2)).T + np.abs(I(L.p_b2))
        assert z_abs.max() < 2 ** 24
        # weights are integers exactly representable in bf16
        for t in L.tensors().values():
            if t is not None:
                assert (t.float() == t.float().round()).all()

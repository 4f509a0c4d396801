"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances (BASELINE.json north_star): masks and ids bit-exact except neurons whose oracle
logit lies within 1e-4 of the threshold; outputs rel-L2 <= 1e-3 (plus an internal regression
gate at 1e-5), computed with the oracle fed the GPU's own ids and
mask bits.  Integer-exact layers must match bit for bit.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import ffn as O
from oracle import partition as OP

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


def run_forward(pi, L, x, fused=True):
    """Whole hot path through pi_layer_forward; returns (y, mask bool, ids, n)."""
    B = x.shape[0]
    y = torch.full((B, L.d), float("nan"), device=x.device)
    mask = L.new_mask(B)
    ids = L.new_ids()
    n = torch.full((1,), -1, dtype=torch.int32, device=x.device)
    L.forward(x, y, mask, ids, n)
    torch.cuda.synchronize()
    nn = int(n.item())
    return y.cpu().numpy(), O.unpack_mask(mask.cpu().numpy().view(np.uint32), L.m_local), \
        ids[:nn].cpu().numpy(), nn


def run_steps(pi, L, x):
    """The same path as three ABI calls: pi_predict -> pi_compact -> pi_sparse_ffn."""
    B = x.shape[0]
    mask = L.new_mask(B)
    logits = torch.empty(B, L.m_local, device=x.device)
    ids = L.new_ids()
    n = torch.zeros(1, dtype=torch.int32, device=x.device)
    y = torch.full((B, L.d), float("nan"), device=x.device)
    L.predict(x, mask, logits)
    L.compact(mask, B, ids, n)
    L.sparse_ffn(x, ids, n, mask, y)
    torch.cuda.synchronize()
    nn = int(n.item())
    return (y.cpu().numpy(), O.unpack_mask(mask.cpu().numpy().view(np.uint32), L.m_local),
            ids[:nn].cpu().numpy(), nn, logits.cpu().numpy())


def oracle_check(w, x, y, gmask, gids, norm=False, nid=None, with_bdown=True, tol=TOL, gate=GATE):
    """Checks GPU outputs against the oracle; returns (rel_l2, n_band_flips)."""
    xo = f(x).astype(np.float64)
    if norm:
        xo = O.rms_normalize(xo)
    sel = slice(None) if nid is None else np.asarray(nid)
    p_w2, p_b2 = f(w.p_w2)[sel], (None if w.p_b2 is None else f(w.p_b2)[sel])
    om, z = O.predict(xo, f(w.p_w1), f(w.p_b1), p_w2, p_b2, w.threshold, w.pred_act)
    band = O.near_threshold(z, w.threshold)
    assert ((gmask == om) | band).all(), f"mask mismatch outside band: {np.argwhere((gmask != om) & ~band)[:5]}"
    assert (gids == O.compact(gmask)).all()
    w_up = f(w.w_up)[sel]
    w_gate = None if w.w_gate is None else f(w.w_gate)[sel]
    w_down = f(w.w_down)[:, sel]
    b_up = None if w.b_up is None else f(w.b_up)[sel]
    yo = O.sparse_ffn(xo, gids, gmask, w_up, b_up, w_gate, w_down, f(w.b_down) if with_bdown else None, w.act)
    err = O.rel_l2(y, yo)
    assert err <= tol, f"rel-L2 {err:.3e} > {tol}"
    assert err <= gate, f"rel-L2 {err:.3e} above the internal regression gate {gate}"
    return err, int(((gmask != om) & band).sum())


# ---------------------------------------------------------------------------
# golden worked example (fig:example P:477-505), embedded in d = 8, r = 8 with zero padding
# ---------------------------------------------------------------------------
def _golden_layer(gen, act="relu", b_down=None, dtype=torch.bfloat16):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "fig_example.json")))
    d, m, r = 8, 8, 8

    def pad(a, rows, cols):
        out = torch.zeros(rows, cols)
        a = torch.tensor(a, dtype=torch.float32)
        out[: a.shape[0], : a.shape[1]] = a
        return out

    gate = pad(g["w_up"], m, d)
    up = pad(g["cases"]["G6_reglu"]["w_up_reglu"], m, d) if act == "reglu" else gate
    wdT = pad(g["w_down_T"], m, d)
    cuda = lambda t: t.to(dtype).cuda().contiguous()  # noqa: E731
    w = gen.LayerWeights(d, m, r, act, cuda(up), cuda(gate) if act == "reglu" else None, cuda(wdT.T.contiguous()),
                         None, None if b_down is None else cuda(torch.tensor(b_down + [0] * (d - len(b_down)),
                                                                                dtype=torch.float32)),
                         cuda(pad(g["p_w1"], r, d)), None, cuda(pad(g["p_w2"], m, r)), None,
                         g["threshold"], "relu", None)
    return g, w


def _x8(rows):
    x = torch.zeros(len(rows), 8)
    x[:, :2] = torch.tensor(rows, dtype=torch.float32)
    return x.cuda()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_golden_g1_g2_g3(env, dtype):
    gen, pi = env
    g, w = _golden_layer(gen, dtype=dtype)
    L = pi.Layer(w, max_batch=2)
    y, gm, ids, n, logits = run_steps(pi, L, _x8([[1, 2]]))
    c = g["cases"]
    assert (logits[0] == np.array(c["G1_predict"]["z"][0])).all()
    assert O.pack_mask(gm).tolist() == c["G1_predict"]["mask_words"]
    assert ids.tolist() == c["G1_predict"]["ids"]
    assert (y[0, :2] == np.array(c["G2_sparse_ffn"]["y"][0])).all() and (y[0, 2:] == 0).all()
    y2, gm2, ids2, n2 = run_forward(pi, L, _x8([[1, 2]]))
    assert (y2 == y).all() and ids2.tolist() == [3, 4, 5]
    # G3: all-ones prediction (t = -inf) gives the dense answer
    Lall = pi.Layer(w, max_batch=1, threshold=float("-inf"))
    y3, _, ids3, _ = run_forward(pi, Lall, _x8([[1, 2]]))
    assert ids3.tolist() == list(range(8))
    assert (y3[0, :2] == np.array(c["G3_invariants"]["y_dense"][0])).all()


def test_golden_g4_shards_g5_bias(env):
    gen, pi = env
    g, w = _golden_layer(gen, b_down=[100, 0])
    c = g["cases"]["G4_shards"]
    parts = []
    for k, key in enumerate(("shard_fast", "shard_slow")):
        s = c[key]
        L = pi.Layer(w, neuron_ids=s["neuron_ids"], own_b_down=(k == 0))
        y, gm, ids, n = run_forward(pi, L, _x8([[1, 2]]))
        assert O.pack_mask(gm).tolist() == s["mask_words"]
        assert ids.tolist() == s["local_ids"]
        exp = np.array(s["y"][0], dtype=np.float64) + (np.array([100, 0]) if k == 0 else 0)
        assert (y[0, :2] == exp).all()
        parts.append(y)
    assert (O.merge(parts)[0, :2] == np.array(g["cases"]["G5_b_down"]["y"][0])).all()


def test_golden_g6_reglu_g7_batch(env):
    gen, pi = env
    g, w = _golden_layer(gen, act="reglu")
    L = pi.Layer(w, max_batch=2)
    y, gm, ids, n = run_forward(pi, L, _x8([[1, 2]]))
    assert (y[0, :2] == np.array(g["cases"]["G6_reglu"]["y"][0])).all()
    g, w = _golden_layer(gen)
    L = pi.Layer(w, max_batch=2)
    c = g["cases"]["G7_batch2"]
    y, gm, ids, n = run_forward(pi, L, _x8(c["x"]))
    assert O.pack_mask(gm).tolist() == c["mask_words"]
    assert ids.tolist() == c["union_ids"]
    assert (y[:, :2] == np.array(c["y"])).all()


# ---------------------------------------------------------------------------
# integer-exact layers: bitwise equality, several tiles and ragged tails
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("act,shape", [("relu", (256, 1000, 64)), ("relu", (136, 777, 24)),
                                       ("reglu", (64, 250, 16)), ("reglu", (40, 97, 8))])
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("B", [1, 2, 3, 6, 8])
def test_integer_layers_bitwise(env, act, shape, dtype, B):
    gen, pi = env
    d, m, r = shape
    w = gen.make_int_layer(d, m, r, act, seed=d + m + B, dtype=dtype, device="cuda")
    x = gen.int_tokens(B, d, act, seed=B).cuda()
    L = pi.Layer(w, max_batch=8)
    for runner in ("steps", "fused"):
        if runner == "steps":
            y, gm, ids, n, logits = run_steps(pi, L, x)
        else:
            y, gm, ids, n = run_forward(pi, L, x)
        xo = f(x).astype(np.float64)
        om, z = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), 0.5)
        assert (gm == om).all()
        if runner == "steps":
            assert (logits == z).all()
        assert (ids == O.compact(om)).all() and n == len(O.compact(om))
        yo = O.sparse_ffn(xo, ids, om, f(w.w_up), f(w.b_up), f(w.w_gate), f(w.w_down), f(w.b_down), act)
        assert (y == yo).all(), runner


# ---------------------------------------------------------------------------
# random layers with the configs' shape classes (reduced m for speed), several batches
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,dims", [("c1", (768, 3072, 64)), ("c2", (4096, 2048, 256)),
                                       ("c3", (5120, 1400, 320)), ("c4", (8192, 1024, 512)),
                                       ("c5", (12288, 520, 768))])
@pytest.mark.parametrize("B", [1, 2, 4, 8])
def test_random_layers(env, name, dims, B):
    gen, pi = env
    cfg = gen.CONFIGS[name]
    d, m, r = dims
    w = gen.make_layer(cfg, seed=7, device="cuda", d=d, m=m, r=r)
    flags = pi.PI_FLAG_INPUT_RMSNORM if cfg.rmsnorm else 0
    L = pi.Layer(w, max_batch=8, flags=flags)
    x = gen.tokens(B, d, seed=11, device="cuda") * (3.0 if cfg.rmsnorm else 1.0)
    y, gm, ids, n = run_forward(pi, L, x)
    oracle_check(w, x, y, gm, ids, norm=cfg.rmsnorm)
    y2, gm2, ids2, n2, _ = run_steps(pi, L, x)
    oracle_check(w, x, y2, gm2, ids2, norm=cfg.rmsnorm)
    # the fused kernel and the per-step kernels agree except on near-threshold logits
    xo = O.rms_normalize(f(x)) if cfg.rmsnorm else f(x)
    _, z = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), w.threshold)
    assert ((gm2 == gm) | O.near_threshold(z, w.threshold)).all()
    Lm = pi.Layer(w, max_batch=8, flags=flags | pi.PI_FLAG_MULTI_KERNEL)
    y3, gm3, ids3, n3 = run_forward(pi, Lm, x)
    assert (gm3 == gm2).all() and (y3 == y2).all()   # multi-kernel forward == the three ABI calls


@pytest.mark.parametrize("B", [1, 2, 8])
def test_mode_t_masks_compact_and_ffn(env, B):
    """Bernoulli masks (mode T) fed straight to pi_compact and pi_sparse_ffn."""
    gen, pi = env
    cfg = gen.CONFIGS["c4"]
    d, m, r = 2048, 4000, 64
    w = gen.make_layer(cfg, seed=3, device="cuda", d=d, m=m, r=r)
    L = pi.Layer(w, max_batch=8)
    mk = gen.bernoulli_masks(gen.activity_profile(m, 0.1, seed=3), B, seed=4)
    words = gen.pack_bits(mk).cuda()
    ids = L.new_ids()
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.compact(words, B, ids, n)
    x = gen.tokens(B, d, seed=5, device="cuda")
    y = torch.empty(B, d, device="cuda")
    L.sparse_ffn(x, ids, n, words, y)
    torch.cuda.synchronize()
    nn = int(n.item())
    gids = ids[:nn].cpu().numpy()
    assert (gids == O.compact(mk.numpy())).all()
    yo = O.sparse_ffn(f(x), gids, mk.numpy(), f(w.w_up), None, None, f(w.w_down), None, "relu")
    assert O.rel_l2(y.cpu().numpy(), yo) <= GATE


# ---------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------
def test_empty_mask_gives_bias_or_zero(env):
    gen, pi = env
    for name in ("c1", "c4"):
        cfg = gen.CONFIGS[name]
        w = gen.make_layer(cfg, seed=1, device="cuda", d=512, m=700, r=32)
        L = pi.Layer(w, max_batch=4, threshold=float("inf"))
        x = gen.tokens(3, 512, device="cuda")
        y, gm, ids, n = run_forward(pi, L, x)
        assert n == 0 and not gm.any()
        exp = np.zeros((3, 512)) if w.b_down is None else np.tile(f(w.b_down), (3, 1))
        assert (y == exp).all()
        y2, *_ = run_steps(pi, L, x)
        assert (y2 == exp).all()


def test_full_mask_equals_dense(env):
    gen, pi = env
    cfg = gen.CONFIGS["c2"]
    w = gen.make_layer(cfg, seed=2, device="cuda", d=1024, m=2500, r=64)
    L = pi.Layer(w, max_batch=2, threshold=float("-inf"))
    x = gen.tokens(2, 1024, device="cuda")
    y, gm, ids, n = run_forward(pi, L, x)
    assert n == 2500 and gm.all()
    yd = O.dense_ffn(f(x), f(w.w_up), f(w.b_up), None, f(w.w_down), f(w.b_down))
    assert O.rel_l2(y, yd) <= GATE


def test_nan_logits_inactive(env):
    gen, pi = env
    cfg = gen.CONFIGS["c1"]
    w = gen.make_layer(cfg, seed=2, device="cuda", d=256, m=300, r=32)
    w.p_b2[5] = float("nan")
    w.p_b2[77] = float("inf")
    L = pi.Layer(w, max_batch=1, threshold=float("-inf"))
    y, gm, ids, n = run_forward(pi, L, gen.tokens(1, 256, device="cuda"))
    assert not gm[0, 5] and gm[0, 77] and n == 299


def test_determinism_bitwise(env):
    gen, pi = env
    cfg = gen.CONFIGS["c3"]
    w = gen.make_layer(cfg, seed=9, device="cuda", d=2048, m=4096, r=128)
    L = pi.Layer(w, max_batch=8, flags=pi.PI_FLAG_INPUT_RMSNORM)
    x = gen.tokens(8, 2048, device="cuda")
    ref = run_forward(pi, L, x)[0]
    for _ in range(20):
        assert (run_forward(pi, L, x)[0] == ref).all()


def test_batch_invariance(env):
    """Batched result == each token alone (per-token masks; reading R9)."""
    gen, pi = env
    cfg = gen.CONFIGS["c3"]
    w = gen.make_layer(cfg, seed=4, device="cuda", d=1024, m=2000, r=64)
    L = pi.Layer(w, max_batch=8, flags=pi.PI_FLAG_INPUT_RMSNORM)
    x = gen.tokens(8, 1024, device="cuda")
    y, gm, ids, n = run_forward(pi, L, x)
    for b in (0, 5, 7):
        yb, gmb, idsb, nb = run_forward(pi, L, x[b:b + 1].contiguous())
        assert (gmb[0] == gm[b]).all()
        assert O.rel_l2(yb[0], y[b]) <= GATE


def test_host_path_equals_device_path(env):
    gen, pi = env
    cfg = gen.CONFIGS["c2"]
    w = gen.make_layer(cfg, seed=5, device="cuda", d=1024, m=4096, r=64)
    L = pi.Layer(w, max_batch=4)
    x = gen.tokens(4, 1024, device="cuda")
    yd = run_forward(pi, L, x)[0]
    xh = x.cpu().pin_memory()
    yh = torch.empty(4, 1024).pin_memory()
    L.forward_host(xh, yh)
    assert (yh.numpy() == yd).all()


def test_stack_equals_chained_layers(env):
    gen, pi = env
    cfg = gen.CONFIGS["c4"]
    d, m, r = 1024, 3000, 64
    ws = [gen.make_layer(cfg, layer=l, seed=1, device="cuda", d=d, m=m, r=r) for l in range(3)]
    Ls = [pi.Layer(w, max_batch=2, flags=pi.PI_FLAG_INPUT_RMSNORM, layer_id=l) for l, w in enumerate(ws)]
    x = gen.tokens(2, d, device="cuda")
    y = torch.empty(2, d, device="cuda")
    pi.pi_stack_forward(Ls, x, y)
    cur = x
    for l, L in enumerate(Ls):
        yl, gm, ids, n = run_forward(pi, L, cur)
        oracle_check(ws[l], cur, yl, gm, ids, norm=True)   # per layer on the GPU's own input (R20)
        cur = torch.from_numpy(yl).cuda()
    assert (y.cpu().numpy() == cur.cpu().numpy()).all()


def test_sharded_emulation_merge(env):
    """G shards on one GPU (pi_partition placement, b_down on shard 0): the merged partials equal
    the unsharded result (O5)."""
    gen, pi = env
    cfg = gen.CONFIGS["c5"]
    d, m, r = 1024, 4096, 64
    w = gen.make_layer(cfg, seed=8, device="cuda", d=d, m=m, r=r)
    x = gen.tokens(1, d, device="cuda")
    L = pi.Layer(w)
    y_full, gm_full, ids_full, _ = run_forward(pi, L, x)
    for G in (2, 4, 8):
        owner, sids, off = pi.pi_partition(w.p.astype(np.float32), G, 64)
        parts = []
        for g in range(G):
            nid = sids[off[g]:off[g + 1]]
            Lg = pi.Layer(w, neuron_ids=nid, own_b_down=(g == 0))
            yg, gmg, idsg, ng = run_forward(pi, Lg, x)
            oracle_check(w, x, yg, gmg, idsg, nid=nid, with_bdown=(g == 0))
            assert (gmg[0] == gm_full[0][nid]).all()
            parts.append(yg)
        assert O.rel_l2(O.merge(parts), y_full) <= GATE


def test_partition_then_shard_cover(env):
    gen, pi = env
    p = gen.activity_profile(32768, 0.1, seed=0).astype(np.float32)
    owner, sids, off = pi.pi_partition(p, 8, 64)
    OP.check_partition(owner.tolist(), sids.tolist(), off.tolist(), 32768, 8, 64)


def test_error_paths(env):
    gen, pi = env
    cfg = gen.CONFIGS["c1"]
    w = gen.make_layer(cfg, seed=1, device="cuda", d=256, m=512, r=32)
    L = pi.Layer(w, max_batch=2)
    x = gen.tokens(3, 256, device="cuda")
    with pytest.raises(pi.PiError) as e:
        L.forward(x, torch.empty(3, 256, device="cuda"))
    assert e.value.name == "PI_ERR_INVALID_ARGUMENT"
    xb = torch.zeros(2 * 256 + 1, device="cuda")[1:].view(2, 256)
    with pytest.raises(pi.PiError) as e:
        L.forward(xb, torch.empty(2, 256, device="cuda"))
    assert e.value.name == "PI_ERR_ALIGNMENT"
    with pytest.raises(pi.PiError) as e:
        L.sparse_ffn(x[:2].contiguous(), L.new_ids(), torch.zeros(1, dtype=torch.int32, device="cuda"), None,
                     torch.empty(2, 256, device="cuda"))
    assert e.value.name == "PI_ERR_INVALID_ARGUMENT"


# ---------------------------------------------------------------------------
# full BASELINE sizes, the bench's launch configuration (one layer each; every output checked)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,B", [("c1", 1), ("c2", 1), ("c3", 1), ("c3", 2), ("c3", 4), ("c3", 8), ("c4", 1),
                                    ("c4", 2), ("c5", 1)])
def test_full_size_layers(env, name, B):
    """Full-size layers at the batch sizes the bench lines run (c3: north_star's B = 1-8; B = 2 is
    the fused kernel with x in shared memory, B = 8 the x-stationary per-step up projection)."""
    gen, pi = env
    cfg = gen.CONFIGS[name]
    w = gen.make_layer(cfg, seed=0, device="cuda")
    flags = pi.PI_FLAG_INPUT_RMSNORM if cfg.rmsnorm else 0
    L = pi.Layer(w, max_batch=B, flags=flags)
    x = gen.tokens(B, cfg.d, seed=1, device="cuda")
    y, gm, ids, n = run_forward(pi, L, x)
    err, flips = oracle_check(w, x, y, gm, ids, norm=cfg.rmsnorm)
    act = gm.mean()
    assert 0.03 < act < 0.3, act
    del L, w
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,dims,B", [("c4", (2048, 3000, 64), 1), ("c3", (1024, 2000, 64), 2),
                                         ("c1", (768, 3072, 64), 1), ("c5", (12288, 700, 64), 1),
                                         ("c4", (8192, 32768, 512), 1)])   # full c4 layers: the bench's kernel
def test_stack_kernel_equals_layer_chain(env, name, dims, B):
    """pi_stack_run (one persistent launch for all layers) == chaining pi_layer_forward, bit for bit,
    and every layer matches the oracle on its own input."""
    gen, pi = env
    cfg = gen.CONFIGS[name]
    d, m, r = dims
    flags = pi.PI_FLAG_INPUT_RMSNORM if cfg.rmsnorm else 0
    ws = [gen.make_layer(cfg, layer=l, seed=2, device="cuda", d=d, m=m, r=r) for l in range(4)]
    Ls = [pi.Layer(w, max_batch=2, flags=flags, layer_id=l) for l, w in enumerate(ws)]
    S = pi.StackHandle(Ls)
    x = gen.tokens(B, d, seed=3, device="cuda")
    y = torch.empty(B, d, device="cuda")
    n = torch.zeros(4, dtype=torch.int32, device="cuda")
    S.run(x, y, n)
    torch.cuda.synchronize()
    cur = x
    for l, L in enumerate(Ls):
        yl, gm, ids, nl = run_forward(pi, L, cur)
        assert nl == int(n[l].item())
        oracle_check(ws[l], cur, yl, gm, ids, norm=cfg.rmsnorm)
        cur = torch.from_numpy(yl).cuda()
    assert (y.cpu().numpy() == cur.cpu().numpy()).all()
    # the host-buffer entry point returns the same
    yh = torch.empty(B, d).pin_memory()
    S.run_host(x.cpu().pin_memory(), yh)
    assert (yh.numpy() == y.cpu().numpy()).all()
    # repeated runs are bitwise identical (fixed reduction order)
    for _ in range(3):
        y2 = torch.empty_like(y)
        S.run(x, y2)
        torch.cuda.synchronize()
        assert torch.equal(y2, y)
    S.close()


def test_hot_neuron_prefetch_changes_nothing(env):
    """Hot neurons (neuron_freq / hot_freq, Insight-1) only move data and reorder each CTA's FFN
    share (prefetched hot neurons first): every layer's union count is unchanged and the stack
    output equals the prefetch-off output to fp32 summation order."""
    gen, pi = env
    cfg = gen.CONFIGS["c4"]
    d, m, r = 2048, 4096, 64
    flags = pi.PI_FLAG_INPUT_RMSNORM if cfg.rmsnorm else 0
    ws = [gen.make_layer(cfg, layer=l, seed=5, device="cuda", d=d, m=m, r=r) for l in range(3)]
    x = gen.tokens(1, d, seed=6, device="cuda")
    outs, counts = [], []
    for hot in (None, 0.5):
        Ls = [pi.Layer(w, max_batch=1, flags=flags, layer_id=l,
                       neuron_freq=None if hot is None else w.p, hot_freq=hot if hot else 0.9)
              for l, w in enumerate(ws)]
        S = pi.StackHandle(Ls)
        y = torch.empty(1, d, device="cuda")
        n = torch.zeros(3, dtype=torch.int32, device="cuda")
        for _ in range(3):
            S.run(x, y, n)
        torch.cuda.synchronize()
        outs.append(y.clone())
        counts.append(n.clone())
        S.close()
    assert int(counts[0][0]) == int(counts[1][0])
    assert O.rel_l2(f(outs[1]), f(outs[0]).astype(np.float64)) <= 1e-5


@pytest.mark.parametrize("B", [1, 2])
def test_hot_first_order_integer_bitwise(env, B):
    """Integer-exact layer with most neurons hot (hot-first FFN order, hot_cap 1000): y equals the
    oracle bit for bit and ids_out is still the ascending union."""
    gen, pi = env
    d, m, r = 256, 1000, 64
    w = gen.make_int_layer(d, m, r, "relu", seed=9, dtype="bf16", device="cuda")
    freq = np.linspace(1.0, 0.0, m).astype(np.float32)       # neurons 0..~700 are "hot" at 0.3
    L = pi.Layer(w, max_batch=2, neuron_freq=freq, hot_freq=0.3, hot_cap=1000)
    x = gen.int_tokens(B, d, "relu", seed=B + 3).cuda()
    y, gm, ids, n = run_forward(pi, L, x)
    xo = f(x).astype(np.float64)
    om, _ = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), 0.5)
    assert (gm == om).all()
    assert (ids == O.compact(om)).all()
    yo = O.sparse_ffn(xo, ids, om, f(w.w_up), f(w.b_up), f(w.w_gate), f(w.w_down), f(w.b_down), "relu")
    assert (y == yo).all()


def test_cuda_graph_capture_replay(env):
    """pi_stack_run, pi_layer_forward (fused) and the per-step path (PI_FLAG_MULTI_KERNEL) are
    stream-ordered and capturable: a captured CUDA graph replays to the eager result bit for bit,
    including for a new token written into the captured input buffer (include/pi.h)."""
    gen, pi = env
    from paper_2312_12456_b200.stack import build_stack
    cfg = gen.CONFIGS["c4"]
    dims = {"d": 2048, "m": 4096, "r": 64}
    st, _ = build_stack(cfg, n_layers=3, seed=3, device="cuda", max_batch=2, dims=dims)
    x = gen.tokens(2, 2048, seed=1, device="cuda")
    y = torch.empty_like(x)
    g = st.capture(x, y)
    for tok in range(3):
        x.copy_(gen.tokens(2, 2048, seed=1, step=tok, device="cuda"))
        y_eager = torch.empty_like(y)
        st.step(x, y_eager)
        y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, y_eager), tok
    st.close()
    w = gen.make_layer(cfg, seed=4, device="cuda", **dims)
    for flags in (0, pi.PI_FLAG_MULTI_KERNEL):
        L = pi.Layer(w, max_batch=2, flags=flags)
        x = gen.tokens(2, 2048, seed=2, device="cuda")
        y = torch.empty_like(x)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            L.forward(x, y)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        ref = y.clone()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            L.forward(x, y)
        y.fill_(float("nan"))
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, ref), flags
        L.close()


def test_full_size_c4_stack_bench_configuration(env):
    """The bench's exact launch configuration at full c4 size: 4 layers of d 8192, m 32768, r 512 with
    the hot-neuron L2 prefetch on (planted profile as neuron_freq, hot_freq 0.99, cap 512).  Equal to
    the same stack with the prefetch off to fp32 summation order (the hot neurons go first in each
    CTA's share), and every layer matches the oracle on its own GPU input (R20)."""
    gen, pi = env
    from paper_2312_12456_b200.stack import build_stack
    cfg = gen.CONFIGS["c4"]
    x = gen.tokens(1, cfg.d, seed=7, device="cuda")
    outs = []
    for hot in (0.99, None):
        st, kept = build_stack(cfg, n_layers=4, seed=0, device="cuda", max_batch=1, keep_weights=(hot is not None),
                               hot_freq=hot, hot_cap=512)
        y = torch.empty_like(x)
        st.step(x, y)
        torch.cuda.synchronize()
        outs.append(y.clone())
        if hot is not None:
            assert st.layers[0].info.launches_per_forward == 1
            cur = x
            for l, (w, _) in enumerate(kept):
                yl, gm, ids, nl = run_forward(pi, st.layers[l], cur)
                oracle_check(w, cur, yl, gm, ids, norm=cfg.rmsnorm)
                cur = torch.from_numpy(yl).cuda()
            assert torch.equal(cur, y)
            del kept
        st.close()
        torch.cuda.empty_cache()
    assert O.rel_l2(f(outs[0]), f(outs[1]).astype(np.float64)) <= 1e-5


# ---------------------------------------------------------------------------
# speculative hot prefix (pi_layer_desc.spec_freq; stack launches)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("B", [1, 2])
@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_speculative_prefix_integer_bitwise(env, B, act):
    """Integer-exact layer through a one-layer stack launch with ~40% of the neurons speculative --
    many of them predicted inactive, so the correction path runs -- equals the oracle bit for bit
    (add-then-subtract is exact on integers)."""
    gen, pi = env
    d, m, r = (256, 1000, 64) if act == "relu" else (64, 250, 16)
    w = gen.make_int_layer(d, m, r, act, seed=d + m + B + 3, dtype="bf16", device="cuda")
    freq = np.random.default_rng(B).random(m).astype(np.float32)
    L = pi.Layer(w, max_batch=2, neuron_freq=freq, spec_freq=0.6, hot_freq=2.0)
    assert L.info.n_spec > 0
    S = pi.StackHandle([L])
    x = gen.int_tokens(B, d, act, seed=B + 7).cuda()
    y = torch.empty(B, d, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    S.run(x, y, n)
    torch.cuda.synchronize()
    xo = f(x).astype(np.float64)
    om, z = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), 0.5)
    ids = O.compact(om)
    assert int(n.item()) == len(ids)                 # the union count includes the speculative neurons
    spec = freq >= 0.6
    assert (spec & ~om.any(axis=0)).sum() > 10       # corrections were exercised
    yo = O.sparse_ffn(xo, ids, om, f(w.w_up), f(w.b_up), f(w.w_gate), f(w.w_down), f(w.b_down), act)
    assert (y.cpu().numpy() == yo).all()
    S.close()


@pytest.mark.parametrize("name,dims,B", [("c4", (2048, 4096, 64), 1), ("c3", (1024, 2000, 64), 2),
                                         ("c4", (8192, 32768, 512), 1)])
def test_speculative_prefix_stack_matches(env, name, dims, B):
    """Random layers (planted profile as neuron_freq, spec_freq 0.99 as in the bench): the stack with
    the speculative prefix equals the stack without it up to fp32 summation order, and both equal
    the layer chain's oracle check (per layer on the GPU's own input, R20)."""
    gen, pi = env
    from paper_2312_12456_b200.stack import build_stack
    cfg = gen.CONFIGS[name]
    dd = {"d": dims[0], "m": dims[1], "r": dims[2]}
    x = gen.tokens(B, dims[0], seed=3, device="cuda")
    outs = []
    for spec in (0.0, 0.99):
        st, kept = build_stack(cfg, n_layers=4, seed=2, device="cuda", max_batch=2, keep_weights=(spec > 0),
                               dims=dd, hot_freq=0.9, spec_freq=spec)
        if spec > 0:
            assert st.layers[0].info.n_spec > 0
        y = torch.empty(B, dims[0], device="cuda")
        st.step(x, y)
        torch.cuda.synchronize()
        for _ in range(3):   # deterministic run to run
            y2 = torch.empty_like(y)
            st.step(x, y2)
            torch.cuda.synchronize()
            assert torch.equal(y2, y)
        outs.append(y.cpu().numpy())
        if spec > 0:
            cur = x
            for l, (w, _) in enumerate(kept):
                yl, gm, ids, nl = run_forward(pi, st.layers[l], cur)   # single-layer launches: unspeculated
                oracle_check(w, cur, yl, gm, ids, norm=cfg.rmsnorm)
                cur = torch.from_numpy(yl).cuda()
            assert O.rel_l2(outs[-1], cur.cpu().numpy()) <= GATE
            del kept
        st.close()
        torch.cuda.empty_cache()
    assert O.rel_l2(outs[1], outs[0]) <= GATE

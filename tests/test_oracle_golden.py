"""Pins the oracle to the paper's worked example (fig:example) and SPEC's examples.

Fixture values are the hand-derived small integers in tests/golden/*.json (see the
citation field there).  Everything here must hold exactly (==).
"""
import numpy as np
import pytest

from oracle import ffn as O

pytestmark = pytest.mark.filterwarnings("ignore")


def _layer(g):
    w_up = np.array(g["w_up"], dtype=np.float64)
    p_w1 = np.array(g["p_w1"], dtype=np.float64)
    p_w2 = np.array(g["p_w2"], dtype=np.float64)
    w_down = np.array(g["w_down_T"], dtype=np.float64).T.copy()   # [d, m]
    return w_up, p_w1, p_w2, w_down


def test_g1_predict(golden):
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G1_predict"]
    mask, z = O.predict(c["x"], p_w1, None, p_w2, None, golden["threshold"], "relu")
    assert (z == np.array(c["z"])).all()
    assert (O.pack_mask(mask) == np.array(c["mask_words"], dtype=np.uint32)).all()
    assert O.compact(mask).tolist() == c["ids"]


def test_g2_sparse_ffn(golden):
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G2_sparse_ffn"]
    mask, _ = O.predict(c["x"], p_w1, None, p_w2, None, golden["threshold"])
    ids = O.compact(mask)
    h = O.sparse_hidden(c["x"], ids, mask, w_up, None, None, "relu")
    assert (h == np.array(c["h_at_ids"])).all()
    y = O.sparse_ffn(c["x"], ids, mask, w_up, None, None, w_down, None, "relu")
    assert (y == np.array(c["y"])).all()


def test_g3_exact_mask_and_dense(golden):
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G3_invariants"]
    em = O.exact_mask(c["x"], w_up, None, None, "relu")
    assert O.compact(em).tolist() == c["exact_ids"]
    y_exact = O.sparse_ffn(c["x"], O.compact(em), em, w_up, None, None, w_down, None)
    y_dense = O.dense_ffn(c["x"], w_up, None, None, w_down, None)
    y_all = O.sparse_ffn(c["x"], np.arange(8), None, w_up, None, None, w_down, None)
    assert (y_exact == np.array(c["y_dense"])).all()
    assert (y_dense == np.array(c["y_dense"])).all()
    assert (y_all == np.array(c["y_dense"])).all()
    # the predicted mask misses neuron 7 (false negative): the gap is exactly its term
    mask, _ = O.predict(c["x"], p_w1, None, p_w2, None, golden["threshold"])
    y_pred = O.sparse_ffn(c["x"], O.compact(mask), mask, w_up, None, None, w_down, None)
    assert (y_dense - y_pred == np.array(c["gap"])).all()
    assert (np.array(c["gap"]) == 5 * w_down[:, c["false_negative"]]).all()


def test_g4_shards_merge(golden):
    """fig:example: fast unit holds {3,5,7}, slow unit the rest; predicted {3,4,5};
    fast computes 3 and 5, slow computes 4, 7 skipped; the add merges."""
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G4_shards"]
    parts = []
    for key in ("shard_fast", "shard_slow"):
        s = c[key]
        nid = np.array(s["neuron_ids"])
        mask, _ = O.predict(c["x"], p_w1, None, p_w2[nid], None, golden["threshold"])
        assert (O.pack_mask(mask) == np.array(s["mask_words"], dtype=np.uint32)).all()
        lids = O.compact(mask)
        assert lids.tolist() == s["local_ids"]
        y = O.sparse_ffn(c["x"], lids, mask, w_up[nid], None, None, w_down[:, nid], None)
        assert (y == np.array(s["y"])).all()
        parts.append(y)
    assert (O.merge(parts) == np.array(c["y_merged"])).all()


def test_g5_b_down(golden):
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G5_b_down"]
    mask, _ = O.predict(c["x"], p_w1, None, p_w2, None, golden["threshold"])
    y = O.sparse_ffn(c["x"], O.compact(mask), mask, w_up, None, None, w_down, np.array(c["b_down"]))
    assert (y == np.array(c["y"])).all()


def test_g6_reglu(golden):
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G6_reglu"]
    up = np.array(c["w_up_reglu"], dtype=np.float64)
    mask, _ = O.predict(c["x"], p_w1, None, p_w2, None, golden["threshold"])
    ids = O.compact(mask)
    h = O.sparse_hidden(c["x"], ids, mask, up, None, w_up, "reglu")
    assert (h == np.array(c["h_at_ids"])).all()
    y = O.sparse_ffn(c["x"], ids, mask, up, None, w_up, w_down, None, "reglu")
    assert (y == np.array(c["y"])).all()


def test_g7_batch_per_token_semantics(golden):
    w_up, p_w1, p_w2, w_down = _layer(golden)
    c = golden["cases"]["G7_batch2"]
    mask, z = O.predict(c["x"], p_w1, None, p_w2, None, golden["threshold"])
    assert (z[1] == np.array(c["z2"])).all()
    assert (O.pack_mask(mask) == np.array(c["mask_words"], dtype=np.uint32)).all()
    ids = O.compact(mask)
    assert ids.tolist() == c["union_ids"]
    y = O.sparse_ffn(c["x"], ids, mask, w_up, None, None, w_down, None)
    assert (y == np.array(c["y"])).all()
    # union semantics (ignoring token 2's own bits) would give a different, wrong answer
    y_union = O.sparse_ffn(c["x"], ids, None, w_up, None, None, w_down, None)
    assert (y_union[1] == np.array(c["y_if_union_semantics_token2"])).all()
    # batched == each token alone (batch-composition invariance, reading R9)
    for b in range(2):
        mb, _ = O.predict([c["x"][b]], p_w1, None, p_w2, None, golden["threshold"])
        yb = O.sparse_ffn([c["x"][b]], O.compact(mb), mb, w_up, None, None, w_down, None)
        assert (yb[0] == y[b]).all()


def test_spec_dense_example(spec_examples):
    e = spec_examples["dense_relu_2x2"]
    fc1 = np.array(e["fc1"], dtype=np.float64)
    fc2 = np.array(e["fc2"], dtype=np.float64)
    em = O.exact_mask([e["x"]], fc1, None, None, "relu")
    assert O.compact(em).tolist() == e["mask"]
    assert (O.sparse_hidden([e["x"]], [0, 1], None, fc1, None, None)[0] == np.array(e["h"])).all()
    assert (O.dense_ffn([e["x"]], fc1, None, None, fc2, None)[0] == np.array(e["y"])).all()


def test_spec_merge_examples(spec_examples):
    for k in ("merge_identity", "merge_simple"):
        e = spec_examples[k]
        assert (O.merge([e["a"], e["b"]]) == np.array(e["sum"])).all()


def test_spec_zero_input_and_empty_mask():
    """S:56 zero input -> empty mask, zero output; S:64/S:73 empty set -> zero; empty with b_down -> b_down."""
    rng = np.random.default_rng(0)
    w_up = rng.standard_normal((16, 8))
    w_down = rng.standard_normal((8, 16))
    x = np.zeros((1, 8))
    em = O.exact_mask(x, w_up, None, None)
    assert O.compact(em).size == 0
    assert (O.dense_ffn(x, w_up, None, None, w_down, None) == 0).all()
    y = O.sparse_ffn(rng.standard_normal((1, 8)), [], None, w_up, None, None, w_down, None)
    assert (y == 0).all()
    bd = rng.standard_normal(8)
    y = O.sparse_ffn(rng.standard_normal((1, 8)), [], None, w_up, None, None, w_down, bd)
    assert (y[0] == bd).all()


def test_spec_single_neuron_unit_basis():
    """a single active neuron with h_i = 1 gives exactly column i of FC2."""
    d, m = 6, 10
    rng = np.random.default_rng(1)
    w_down = rng.standard_normal((d, m))
    w_up = np.zeros((m, d))
    x = np.zeros((1, d))
    x[0, 0] = 1.0
    w_up[4, 0] = 1.0                          # a_4 = 1 -> h_4 = 1
    y = O.sparse_ffn(x, [4], None, w_up, None, None, w_down, None)
    assert (y[0] == w_down[:, 4]).all()

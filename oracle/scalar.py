"""Scalar brute-force twin of oracle/ffn.py for tiny layers (pure Python loops).

TEST INFRASTRUCTURE ONLY (see oracle/ffn.py header).

Written directly from the textbook definition of the layer (P:177-205
fig:bg-mlp) with explicit loops over single floats, so it shares no
vectorised code with ffn.py.  Used only on tiny shapes (d <= 8, m <= 16) to pin
ffn.py against an independent computation.
"""
from __future__ import annotations


def predict(x, p_w1, p_b1, p_w2, p_b2, t, pred_act="relu"):
    r = len(p_w1)
    d = len(x)
    g = []
    for j in range(r):
        s = 0.0
        for k in range(d):
            s += float(p_w1[j][k]) * float(x[k])
        if p_b1 is not None:
            s += float(p_b1[j])
        g.append(max(s, 0.0) if pred_act == "relu" else s)
    out = []
    for i in range(len(p_w2)):
        s = 0.0
        for j in range(r):
            s += float(p_w2[i][j]) * g[j]
        if p_b2 is not None:
            s += float(p_b2[i])
        out.append(s > t)
    return out


def ffn_masked(x, active, w_up, b_up, w_gate, w_down, b_down, act="relu"):
    """y = b_down + sum_{i active} act_i(x) * W_down[:, i] for ONE token (active: list of bool)."""
    d = len(x)
    m = len(w_up)
    y = [float(b_down[j]) if b_down is not None else 0.0 for j in range(d)]
    for i in range(m):
        if not active[i]:
            continue
        a = 0.0
        for k in range(d):
            a += float(w_up[i][k]) * float(x[k])
        if b_up is not None:
            a += float(b_up[i])
        if act == "relu":
            h = a if a > 0.0 else 0.0
        else:
            gt = 0.0
            for k in range(d):
                gt += float(w_gate[i][k]) * float(x[k])
            h = (gt if gt > 0.0 else 0.0) * a
        for j in range(d):
            y[j] += h * float(w_down[j][i])
    return y

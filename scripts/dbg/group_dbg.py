import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2312_12456_b200 import gen, pi
from oracle import ffn as O
mode, pg, ng, d, m, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
torch.cuda.set_device(0)
ws = [gen.make_int_layer(d, m, r, "relu", seed=17 * k + d, dtype="bf16", device="cuda") for k in range(ng)]
Ls = [pi.Layer(w, max_batch=1) for w in ws]
x = torch.stack([gen.int_tokens(1, d, "relu", seed=k).cuda() for k in range(ng)])
y = torch.full((ng, 1, d), float("nan"), device="cuda")
n = torch.full((ng, 1), -1, dtype=torch.int32, device="cuda")
if mode == "layer":
    for k in range(ng):
        Ls[k].forward(x[k], y[k], None, None, n[k])
else:
    G = pi.GroupHandle([[L] for L in Ls], pg)
    G.run(x, y, n)
torch.cuda.synchronize()
ok = True
for k, w in enumerate(ws):
    xo = x[k].cpu().numpy().astype(np.float64)
    f = lambda t: None if t is None else t.float().cpu().numpy()
    om, _ = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), 0.5)
    ids = O.compact(om)
    yo = O.sparse_ffn(xo, ids, om, f(w.w_up), f(w.b_up), f(w.w_gate), f(w.w_down), f(w.b_down), "relu")
    ok &= int(n[k, 0]) == len(ids) and bool((y[k].cpu().numpy() == yo).all())
print(mode, pg, ng, d, m, r, "OK" if ok else "MISMATCH", int(n[0, 0]))

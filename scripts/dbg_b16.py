import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import ffn as O
from paper_2312_12456_b200 import gen, pi
torch.cuda.set_device(0)
d, m, r = 256, 1000, 64
for B in (9, 12, 16, 24, 32):
  for dtype in ("bf16",):
    w = gen.make_int_layer(d, m, r, "relu", seed=d + m + 16, dtype=dtype, device="cuda")
    L = pi.Layer(w, max_batch=32)
    x = gen.int_tokens(B, d, "relu", seed=16).cuda()
    mask = L.new_mask(B); logits = torch.empty(B, m, device="cuda")
    L.predict(x, mask, logits); torch.cuda.synchronize()
    xo = x.double().cpu().numpy()
    f = lambda t: None if t is None else t.float().cpu().numpy()
    om, z = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), 0.5)
    gz = logits.cpu().numpy()
    bad = np.argwhere(gz != z)
    print(B, dtype, "logit mismatches", len(bad), "tokens", sorted(set(bad[:,0].tolist()))[:20], "first", bad[:3].tolist(), [ (gz[i,j], z[i,j]) for i,j in bad[:3]])
    # g
    g = L.__dict__.get('g')

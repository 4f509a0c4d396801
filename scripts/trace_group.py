# Phase trace of group 0 of a grouped launch (pi_group_run): python scripts/trace_group.py c2 8 18 3  (config, CTAs per group, groups, layers per group)
import sys, torch, numpy as np, json
sys.path.insert(0, '.')
from paper_2312_12456_b200 import gen, pi
from paper_2312_12456_b200.stack import build_stack
name, pg, ng, gl = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
torch.cuda.set_device(0)
cfg = gen.CONFIGS[name]
stacks = [build_stack(cfg, n_layers=gl, seed=100 * k, device="cuda", max_batch=1)[0] for k in range(ng)]
G = pi.GroupHandle([st.layers for st in stacks], pg)
d = cfg.d
x = torch.stack([gen.tokens(1, d, seed=k, device="cuda") for k in range(ng)])
y = torch.empty(ng, 1, d, device="cuda")
for _ in range(3): G.run(x, y)
buf = torch.zeros(148 * 256, dtype=torch.int64, device="cuda")
L0 = stacks[0].layers[0]
L0.set_trace(buf)
G.run(x, y); torch.cuda.synchronize(); L0.set_trace(None)
t = buf.view(148, 256)[:pg].cpu().numpy().astype(np.float64)
rel = (t[:, :9] - t[:, :1]) / 1e3
names = ["start", "P1 done", "bar1", "P2 done", "bar2", "ids", "FFN done", "bar3", "end"]
print(name, "pg", pg, "mean", dict(zip(names, np.round(rel.mean(0), 2))))
print(" max", dict(zip(names, np.round(rel.max(0), 2))))
st = (t[:, 16:72] - t[:, :1]) / 1e3
print(" cta0 stage ready us", np.round(st[0][st[0] > -1e6][:56], 2).tolist())
iss = (t[:, 72:128] - t[:, :1]) / 1e3
print(" cta0 stage issue us", np.round(iss[0][:56], 2).tolist())

"""a6 on the product path: the neuron-sharded multi-rank step (stack.Stack.step, world > 1) run
by real ranks, compared with the oracle and with the unsharded stack.

Each rank is its own process with its own libpi handles for its shard (pi_partition placement,
b_down on rank 0), all on cuda:0 -- this box has one GPU and NCCL refuses two ranks on one
device, so the ranks talk through a gloo process group over CUDA tensors.  Stack.step is the
code the bench runs at N > 1 with NCCL: per layer pi_layer_forward on the local shard, then
all_reduce(SUM) of the fp32 partials (the paper's merge).  Checked:
  * integer-exact layers: the merged output equals the oracle bit for bit (G = 2, 4);
  * random chained layers: every rank holds the same merged output; each layer's merged output
    matches the unsharded oracle on that layer's GPU input (R20) within the north_star
    tolerance; the merged stack equals the unsharded GPU stack (world 1) within the 1e-5 gate;
  * the per-layer union counts of the shards add up to the unsharded count."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import ffn as O

pytestmark = pytest.mark.gpu

TOL = 1e-3
GATE = 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, kind, args):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2312_12456_b200 import gen, pi
        from paper_2312_12456_b200.stack import LayerMeta, Stack, build_stack, shard_ids
        if kind == "int":
            d, m, r, act, B = args
            w = gen.make_int_layer(d, m, r, act, seed=d + m, dtype="bf16", device="cuda")
            nid = shard_ids(np.random.default_rng(m).random(m), world, rank)   # any profile: exact anyway
            L = pi.Layer(w, neuron_ids=nid, max_batch=B, own_b_down=(rank == 0))
            st = Stack([L], [LayerMeta(d, len(nid), r, act == "reglu", True, rank == 0, True, True)], rank, world,
                       dist.group.WORLD)
            x = gen.int_tokens(B, d, act, seed=B).cuda()
        else:
            name, dims, n_layers, B = args
            cfg = gen.CONFIGS[name]
            st, _ = build_stack(cfg, n_layers=n_layers, rank=rank, world=world, seed=4, device="cuda", max_batch=B,
                                group=dist.group.WORLD, dims=dims)
            x = gen.tokens(B, dims["d"], seed=5, device="cuda")
        y = torch.empty_like(x)
        n_out = torch.zeros(len(st), dtype=torch.int32, device="cuda")
        rec = []
        st.step(x, y, n_out, record=rec)
        torch.cuda.synchronize()
        # (gloo collectives are not CUDA-graph capturable; Stack.capture is covered with NCCL / world 1)
        # numpy (pickled by value): torch CPU tensors would travel as shared-memory handles that die
        # with this process
        q.put((rank, {"y": y.cpu().numpy(), "rec": [t.cpu().numpy() for t in rec], "n": n_out.cpu().numpy()}))
        st.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


def _run(world, kind, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, kind, args)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    return res


def f(t):
    return None if t is None else t.float().cpu().numpy()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("act", ["relu", "reglu"])
def test_sharded_step_integer_layer_bitwise(world, act):
    from paper_2312_12456_b200 import gen
    d, m, r, B = (256, 1024, 64, 3) if act == "relu" else (64, 256, 16, 3)
    res = _run(world, "int", (d, m, r, act, B))
    w = gen.make_int_layer(d, m, r, act, seed=d + m, dtype="bf16", device="cpu")
    x = gen.int_tokens(B, d, act, seed=B).double().numpy()
    om, _ = O.predict(x, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), 0.5)
    yo = O.sparse_ffn(x, O.compact(om), om, f(w.w_up), f(w.b_up), f(w.w_gate), f(w.w_down), f(w.b_down), act)
    for rk in range(world):
        assert (res[rk]["y"] == yo).all(), rk
    assert sum(int(res[rk]["n"][0]) for rk in range(world)) == len(O.compact(om))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_random_stack(world):
    from paper_2312_12456_b200 import gen
    from paper_2312_12456_b200.stack import build_stack
    name, dims, n_layers, B = "c4", {"d": 1024, "m": 4096, "r": 64}, 3, 2
    res = _run(world, "rand", (name, dims, n_layers, B))
    y0 = res[0]["y"]
    for rk in range(1, world):
        assert (res[rk]["y"] == y0).all(), "ranks disagree after the all-reduce"
    # unsharded GPU stack (world 1, one persistent launch) on the same weights and token
    cfg = gen.CONFIGS[name]
    st, kept = build_stack(cfg, n_layers=n_layers, seed=4, device="cuda", max_batch=B, keep_weights=True, dims=dims)
    x = gen.tokens(B, dims["d"], seed=5, device="cuda")
    y = torch.empty_like(x)
    n1 = torch.zeros(n_layers, dtype=torch.int32, device="cuda")
    st.step(x, y, n1)
    torch.cuda.synchronize()
    assert O.rel_l2(y0, y.cpu().numpy()) <= GATE
    n_sh = sum(res[rk]["n"] for rk in range(world))
    assert (np.abs(n_sh - n1.cpu().numpy()) <= 2).all(), (n_sh, n1)   # equal up to near-threshold flips
    # each layer's merged output against the unsharded oracle on that layer's GPU input (R20)
    cur = f(x).astype(np.float64)
    for l, (w, _) in enumerate(kept):
        xo = O.rms_normalize(cur) if cfg.rmsnorm else cur
        om, z = O.predict(xo, f(w.p_w1), f(w.p_b1), f(w.p_w2), f(w.p_b2), w.threshold)
        yo = O.sparse_ffn(xo, O.compact(om), om, f(w.w_up), f(w.b_up), f(w.w_gate), f(w.w_down), f(w.b_down), w.act)
        yl = res[0]["rec"][l]
        if not O.near_threshold(z, w.threshold).any():
            err = O.rel_l2(yl, yo)
            assert err <= TOL and err <= GATE, (l, err)
        cur = yl.astype(np.float64)
    st.close()

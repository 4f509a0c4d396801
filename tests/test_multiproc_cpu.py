"""World-size-2 gloo tests of the multi-GPU host logic on CPU.

Each rank takes its neuron shard with the product's placement helper (stack.shard_ids ->
pi_partition), computes its partial output for the shard (the CPU oracle stands in for the
GPU kernels here), and the partials are merged with an all-reduce(sum), exactly as stack.Stack
does with NCCL between layers.  The merged result must equal the unsharded layer, b_down counted
once (P:504-505 merge; fig:example split P:489-505)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import ffn as O
        from paper_2312_12456_b200 import gen
        from paper_2312_12456_b200.stack import shard_ids

        cfg = gen.CONFIGS["c5"]
        ok = True
        for layer in range(2):
            w = gen.make_layer(cfg, layer=layer, seed=5, d=64, m=1024, r=16)
            f = lambda t: None if t is None else t.float().numpy()  # noqa: E731
            x = gen.tokens(2, 64, seed=layer).numpy().astype(np.float64)
            nid = shard_ids(w.p, world, rank)
            assert len(nid) == 1024 // world and (np.diff(nid) > 0).all()
            # local predictor rows + local FFN rows (neuron table = nid)
            mask, _ = O.predict(x, f(w.p_w1), None, f(w.p_w2)[nid], f(w.p_b2)[nid], w.threshold)
            ids = O.compact(mask)
            part = O.sparse_ffn(x, ids, mask, f(w.w_up)[nid], f(w.b_up)[nid], None, f(w.w_down)[:, nid],
                                f(w.b_down) if rank == 0 else None, "relu")
            t = torch.from_numpy(part)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            # unsharded reference
            mk, _ = O.predict(x, f(w.p_w1), None, f(w.p_w2), f(w.p_b2), w.threshold)
            ref = O.sparse_ffn(x, O.compact(mk), mk, f(w.w_up), f(w.b_up), None, f(w.w_down), f(w.b_down), "relu")
            ok &= O.rel_l2(t.numpy(), ref) < 1e-12
            # every neuron owned by exactly one rank
            allids = [None] * world
            dist.all_gather_object(allids, nid.tolist())
            flat = sorted(i for lst in allids for i in lst)
            ok &= flat == list(range(1024))
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.timeout(300)
def test_world2_shard_and_merge():
    from paper_2312_12456_b200 import build
    build.build_lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res

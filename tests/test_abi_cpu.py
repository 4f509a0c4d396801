"""CPU-side checks of the C ABI: the library loads, exports every symbol include/pi.h declares,
pi_partition (host code) matches the oracle bit for bit, and host-side validation rejects bad
arguments before touching the device (fake device pointers are never dereferenced)."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

from oracle import partition as OP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pi():
    from paper_2312_12456_b200 import build
    build.build_lib()
    from paper_2312_12456_b200 import pi as _pi
    return _pi


def _declared():
    src = open(os.path.join(ROOT, "include", "pi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pi_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(pi):
    names = _declared()
    assert len(names) >= 12
    lib = pi.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(pi.EXPORTS)


def test_version(pi):
    assert "sm_100a" in pi.pi_version()


def test_partition_matches_oracle(pi):
    rnd = random.Random(5)
    for trial in range(40):
        G = rnd.choice([1, 2, 3, 4, 8])
        gr = rnd.choice([1, 2, 64]) if trial % 3 else 1
        m = G * gr * rnd.randint(1, 6)
        f = np.array([rnd.random() ** 4 for _ in range(m)], dtype=np.float32)
        if trial % 5 == 0:
            f[: m // 2] = f[0]            # many ties
        owner, ids, off = pi.pi_partition(f, G, gr)
        o2, i2, off2 = OP.partition(f.tolist(), G, gr)
        assert owner.tolist() == o2 and ids.tolist() == i2 and off.tolist() == off2
        OP.check_partition(owner.tolist(), ids.tolist(), off.tolist(), m, G, gr)


def test_partition_paper_scale(pi):
    """m = 32768 neurons, 8 GPUs, 64-neuron runs, power-law impacts."""
    from paper_2312_12456_b200 import gen
    f = gen.activity_profile(32768, 0.1, seed=0).astype(np.float32)
    owner, ids, off = pi.pi_partition(f, 8, 64)
    o2, i2, off2 = OP.partition(f.tolist(), 8, 64)
    assert owner.tolist() == o2 and ids.tolist() == i2
    loads = OP.shard_loads(f.tolist(), owner.tolist(), 8)
    assert max(loads) / (sum(loads) / 8) < 1.01       # expected active mass balanced


def test_partition_errors(pi):
    with pytest.raises(pi.PiError) as e:
        pi.pi_partition(np.ones(10, np.float32), 3, 1)
    assert e.value.name == "PI_ERR_SHAPE"
    with pytest.raises(pi.PiError) as e:
        pi.pi_partition(np.array([1.0, np.nan], np.float32), 2, 1)
    assert e.value.name == "PI_ERR_INVALID_ARGUMENT"
    with pytest.raises(pi.PiError) as e:
        pi.pi_partition(np.ones(8, np.float32), 0, 1)
    assert e.value.name == "PI_ERR_INVALID_ARGUMENT"


def _desc(pi, **kw):
    base = dict(layer_id=7, d=64, m_total=128, rank=16, m_local=128, neuron_ids=None, dtype=1, act=0,
                pred_act=0, w_up=0x10000, w_gate=None, w_down=0x20000, b_up=None, b_down=None, p_w1=0x30000,
                p_b1=None, p_w2=0x40000, p_b2=None, logit_threshold=0.0, max_batch=1, flags=0)
    base.update(kw)
    return pi.LayerDesc(**base)


def _create_status(pi, desc):
    h = ctypes.c_void_p()
    st = pi.lib().pi_layer_create(ctypes.byref(desc), None, ctypes.byref(h))
    return st, pi.lib().pi_last_error().decode(), h


@pytest.mark.parametrize("kw,status", [
    (dict(d=12), 4),                        # d % 8 -> ALIGNMENT
    (dict(rank=12), 4),
    (dict(w_up=0x10004), 4),                # misaligned weight pointer
    (dict(m_local=64), 2),                  # neuron_ids NULL requires m_local == m_total
    (dict(m_local=256), 2),
    (dict(max_batch=33), 1),                # > PI_MAX_BATCH
    (dict(max_batch=9), 5),                 # tensor-core batched path needs d % 128 == 0 -> UNSUPPORTED
    (dict(ffn_format=7), 1),                # unknown FFN format
    (dict(ffn_format=1), 1),                # PI_FFN_Q4 without scales
    (dict(ffn_format=1, d=40, w_up_scale=0x50000, w_down_scale=0x60000), 4),   # Q4 needs d % 32 == 0
    (dict(w_up_scale=0x50000), 1),          # scales only for Q4
    (dict(ffn_format=1, max_batch=16, d=128, w_up_scale=0x50000, w_down_scale=0x60000), 5),  # Q4 is B <= 8
    (dict(max_batch=0), 1),
    (dict(act=1), 1),                       # ReGLU without gate
    (dict(dtype=5), 5),
    (dict(flags=4), 1),
    (dict(logit_threshold=float("nan")), 1),
    (dict(p_w2=None), 1),
])
def test_create_validation(pi, kw, status):
    st, msg, h = _create_status(pi, _desc(pi, **kw))
    assert st == status, msg
    assert h.value is None


def test_create_validation_neuron_ids(pi):
    for ids, status in (([0, 5, 5, 9], 3), ([0, 5, 4, 9], 3), ([0, 1, 2, 128], 3), ([-1, 1, 2, 3], 3)):
        arr = (ctypes.c_int32 * 4)(*ids)
        st, msg, h = _create_status(pi, _desc(pi, m_local=4, neuron_ids=arr))
        assert st == status, msg
        assert "layer 7" in msg


def test_null_handles(pi):
    lib = pi.lib()
    assert lib.pi_layer_create(None, None, None) == 1
    assert lib.pi_layer_destroy(None) == 0
    assert lib.pi_predict(None, None, 1, None, None, None) == 1
    assert lib.pi_compact(None, None, 1, None, None, None) == 1
    assert lib.pi_sparse_ffn(None, None, 1, None, None, None, None, None) == 1
    assert lib.pi_layer_forward(None, None, 1, None, None, None, None, None) == 1
    assert lib.pi_layer_forward_host(None, None, 1, None, None) == 1
    assert lib.pi_stack_forward(None, 0, None, 1, None, None, None) == 1
    assert lib.pi_stack_forward_host(None, 0, None, 1, None, None) == 1
    assert lib.pi_layer_set_trace(None, None) == 1
    assert lib.pi_stack_create(None, 1, None) == 1
    assert lib.pi_stack_destroy(None) == 0
    assert lib.pi_stack_run(None, None, 1, None, None, None) == 1
    assert lib.pi_stack_run_host(None, None, 1, None, None) == 1
    assert "NULL" in lib.pi_last_error().decode()
    assert lib.pi_group_create(None, 1, 1, 1, 0, None) == 1
    assert lib.pi_group_destroy(None) == 0
    assert lib.pi_group_run(None, None, 1, None, None, None) == 1
    assert "NULL" in lib.pi_last_error().decode()

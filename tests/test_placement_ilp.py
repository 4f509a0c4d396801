"""The paper's placement ILP (Eqs. 1-8; row f4).

The brute-force oracle (oracle/placement.py) is pinned to hand-computed instances and to closed
forms (unlimited capacity puts everything on the fast unit; zero capacity nothing; an
uncrossable T_sync nothing; Eq. 4's threshold by hand); then pi_place_ilp (the exact C++ DP) must
reach the oracle's optimum on hundreds of seeded tiny instances, with an assignment that satisfies
Eqs. 3-8 (checked by the oracle's constraint checker)."""
import math
import random

import numpy as np
import pytest

from oracle import placement as OPL


@pytest.fixture(scope="module")
def pi():
    from paper_2312_12456_b200 import build
    build.build_lib()
    from paper_2312_12456_b200 import pi as _pi
    return _pi


def test_min_fast_count_by_hand():
    # T_fast = 0.5, T_slow = 1: C * 0.5 + 1.2 <= C  ->  C >= 2.4  ->  3
    assert OPL.min_fast_count(1, 2.0, 1.0, 1.2) == 3
    assert OPL.min_fast_count(1, 2.0, 1.0, 0.0) == 0
    assert OPL.min_fast_count(4, 4.0, 1.0, 3.0) == 1        # T_fast 1, T_slow 4: C + 3 <= 4 C
    assert OPL.min_fast_count(1, 1.0, 2.0, 0.0) is None     # the fast unit is not faster


def test_hand_instance():
    # two layers of 4 neurons, granule 2, 1 byte per neuron, fast capacity < 5 bytes (so <= 4),
    # T_sync small: layer batches (by -f): L0 {0.9+0.8=1.7, 0.3+0.1=0.4}, L1 {0.6+0.5=1.1, 0.2+0.0}
    f = [[0.9, 0.1, 0.8, 0.3], [0.5, 0.0, 0.6, 0.2]]
    obj, fast = OPL.brute_force(f, [1, 1], 2, 5.0, 2.0, 1.0, 0.1)
    assert math.isclose(obj, 1.7 + 1.1)
    assert fast == [[1, 0, 1, 0], [1, 0, 1, 0]]
    # Eq. 4 needs C_l >= 3 neurons (T_sync 1.2): a layer takes 0 or both batches; capacity 4 -> one layer
    obj, fast = OPL.brute_force(f, [1, 1], 2, 5.0, 2.0, 1.0, 1.2)
    assert math.isclose(obj, 1.7 + 0.4) and fast == [[1, 1, 1, 1], [0, 0, 0, 0]]


def test_closed_forms():
    rng = random.Random(1)
    f = [[rng.random() for _ in range(6)] for _ in range(2)]
    obj, fast = OPL.brute_force(f, [2, 3], 2, math.inf, 3.0, 1.0, 0.0)
    assert math.isclose(obj, sum(map(sum, f))) and all(all(r) for r in fast)
    obj, fast = OPL.brute_force(f, [2, 3], 2, 0.0, 3.0, 1.0, 0.0)
    assert obj == 0.0 and not any(any(r) for r in fast)
    obj, fast = OPL.brute_force(f, [2, 3], 2, math.inf, 3.0, 1.0, 1e9)   # C_l > m: nothing pays off
    assert obj == 0.0


def _instance(seed):
    rng = random.Random(seed)
    L = rng.choice([1, 2, 3])
    m = rng.choice([4, 6, 8])
    granule = rng.choice([1, 2, 3])
    while (m + granule - 1) // granule * L > 14:
        granule += 1
    f = [[round(rng.random() ** 3, 3) for _ in range(m)] for _ in range(L)]
    nbytes = [rng.choice([1, 2, 4]) for _ in range(L)]
    mcap = rng.choice([0.0, 3.0, 7.5, 12.0, 20.0, 1e9])
    bw_fast, bw_slow = rng.choice([(4.0, 1.0), (2.0, 1.0), (1.0, 2.0), (8.0, 1.0)])
    t_sync = rng.choice([0.0, 0.5, 2.0, 6.0])
    return f, nbytes, granule, mcap, bw_fast, bw_slow, t_sync


@pytest.mark.parametrize("seed", range(300))
def test_dp_matches_brute_force(pi, seed):
    f, nbytes, granule, mcap, bwf, bws, ts = _instance(seed)
    obj_o, _ = OPL.brute_force(f, nbytes, granule, mcap, bwf, bws, ts)
    fast, cnt, obj = pi.pi_place_ilp(np.array(f, np.float32), nbytes, granule, mcap, bwf, bws, ts)
    assert math.isclose(obj, obj_o, rel_tol=1e-6, abs_tol=1e-6), (obj, obj_o)
    # the returned assignment is feasible (Eqs. 3-8) and reaches the objective it reports
    f32 = np.array(f, np.float32).astype(np.float64).tolist()
    val = OPL.check_assignment(fast.tolist(), f32, nbytes, granule, mcap, bwf, bws, ts)
    assert math.isclose(val, obj, rel_tol=1e-6, abs_tol=1e-6)
    assert cnt.tolist() == [int(r.sum()) for r in fast]


def test_c4_scale_and_validation(pi):
    """60 layers of a c4-sized profile: the hot tier is the top of each layer (ties by id), the
    per-layer counts are whole batches of 64, and the budget is respected."""
    from paper_2312_12456_b200 import gen
    L, m = 60, 32768
    f = np.stack([gen.activity_profile(m, 0.10, seed=0, layer=l) for l in range(L)]).astype(np.float32)
    nb = [2 * 2 * 8192] * L                    # up + down rows of one neuron, bf16
    fast, cnt, obj = pi.pi_place_ilp(f, nb, 64, 60e6, 20e12, 6.5e12, 0.5e-6)
    assert (cnt % 64 == 0).all() and cnt.sum() * nb[0] < 60e6
    for l in range(L):
        order = np.lexsort((np.arange(m), -f[l]))
        k = cnt[l]
        assert fast[l, order[:k]].all() and not fast[l, order[k:]].any()
    with pytest.raises(pi.PiError):
        pi.pi_place_ilp(np.full((2, 4), np.nan, np.float32), [1, 1], 2, 10.0, 2.0, 1.0, 0.0)
    with pytest.raises(pi.PiError):
        pi.pi_place_ilp(np.ones((2, 4), np.float32), [1.5, 1], 2, 10.0, 2.0, 1.0, 0.0)

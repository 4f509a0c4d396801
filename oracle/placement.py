"""CPU oracle for the paper's neuron-placement ILP.

TEST INFRASTRUCTURE ONLY (see oracle/ffn.py header).

PowerInfer places neurons on a fast unit (GPU) or a slow unit (CPU) by an integer linear program
(P:727-811), written here in the paper's notation:

  Eq. 1  v_i = f_i                                   impact = profiled activation frequency
  Eq. 2  maximise  sum_{e in N} a_{fast,e} v_e       impact placed on the fast unit
  Eq. 3  sum_{i in U} a_{i,n} = 1                    every neuron on exactly one unit
  Eq. 4  C_l T_l^fast + T_sync <= C_l T_l^slow       a layer split between units must put at least
                                                     C_l neurons on the fast unit to pay for the
                                                     synchronisation it causes
  Eq. 5  T_l^j = M_l / Bandwidth_j                   a neuron's time = reading its weights once
  Eq. 6  sum_n a_{j,n} M_n < MCap_j                  memory capacity of each unit (strict)
  Eq. 7  sum_{e in N_l} a_{fast,e} >= C_l y_l        with y_l binary: a layer has either no
  Eq. 8  sum_{e in N_l} a_{fast,e} <= K y_l          neuron on the fast unit or at least C_l

and, to keep the problem tractable, "groups 64 neurons with similar impacts from a layer into a
single batch": each layer's neurons are ordered by (-f_i, i) and cut into consecutive
runs of `granule`; a batch is placed as a whole (its impact is the sum of its neurons' f_i).

Readings (R22): C_l is the smallest neuron count that satisfies Eq. 4 (a layer whose
fast unit is not faster, T_l^fast >= T_l^slow, cannot put anything on the fast unit), rounded up
to whole batches; the slow unit's capacity is unlimited unless given.

This oracle enumerates every assignment of batches to the two units on tiny instances, keeps
the ones satisfying Eqs. 3-8 and returns the best Eq. 2 objective (brute force: it is the
definition, not an algorithm).
"""
from __future__ import annotations

import itertools
import math


def batches(freq_layers, granule):
    """Per layer: list of batches, each a list of neuron ids, in (-f, id) order."""
    out = []
    for f in freq_layers:
        order = sorted(range(len(f)), key=lambda i: (-float(f[i]), i))
        out.append([order[k:k + granule] for k in range(0, len(order), granule)])
    return out


def min_fast_count(neuron_bytes, bw_fast, bw_slow, t_sync):
    """Eq. 4 with Eq. 5: the smallest C with C M / BW_fast + T_sync <= C M / BW_slow, or None."""
    t_fast = neuron_bytes / bw_fast
    t_slow = neuron_bytes / bw_slow
    if t_slow <= t_fast:
        return None
    c = math.ceil(t_sync / (t_slow - t_fast) - 1e-12)
    while c * t_fast + t_sync > c * t_slow:      # guard the floating-point ceiling
        c += 1
    return max(c, 0)


def brute_force(freq_layers, neuron_bytes, granule, mcap_fast, bw_fast, bw_slow, t_sync, mcap_slow=math.inf):
    """Best Eq. 2 objective over all batch assignments satisfying Eqs. 3-8; returns
    (objective, fast flags per layer per neuron) of one optimal assignment."""
    bl = batches(freq_layers, granule)
    flat = [(l, k) for l, lb in enumerate(bl) for k in range(len(lb))]
    cmin = []
    for l in range(len(bl)):
        c = min_fast_count(neuron_bytes[l], bw_fast, bw_slow, t_sync)
        cmin.append(None if c is None else c)
    best, best_sel = -1.0, None
    for sel in itertools.product((0, 1), repeat=len(flat)):        # 1 = fast unit (Eq. 3 by construction)
        mem_fast = mem_slow = 0.0
        count = [0] * len(bl)
        value = 0.0
        for (l, k), a in zip(flat, sel):
            nb = len(bl[l][k])
            if a:
                mem_fast += nb * neuron_bytes[l]
                count[l] += nb
                value += sum(float(freq_layers[l][i]) for i in bl[l][k])
            else:
                mem_slow += nb * neuron_bytes[l]
        # Eq. 6 (strict); a unit holding no neuron satisfies it trivially
        if (mem_fast > 0 and not mem_fast < mcap_fast) or (mem_slow > 0 and not mem_slow < mcap_slow):
            continue
        ok = True
        for l in range(len(bl)):                                    # Eqs. 4, 7, 8
            y = 1 if count[l] > 0 else 0
            if y and (cmin[l] is None or count[l] < cmin[l]):
                ok = False
                break
        if ok and value > best + 1e-12:
            best, best_sel = value, sel
    fast = [[0] * len(f) for f in freq_layers]
    for (l, k), a in zip(flat, best_sel):
        if a:
            for i in bl[l][k]:
                fast[l][i] = 1
    return best, fast


def check_assignment(fast, freq_layers, neuron_bytes, granule, mcap_fast, bw_fast, bw_slow, t_sync):
    """Eqs. 3-8 for a given fast-flag assignment (whole batches); returns its Eq. 2 objective."""
    bl = batches(freq_layers, granule)
    mem = 0.0
    value = 0.0
    for l, lb in enumerate(bl):
        cnt = 0
        for b in lb:
            flags = {fast[l][i] for i in b}
            assert len(flags) == 1, "a batch is split across units (P:808-809)"
            if flags == {1}:
                cnt += len(b)
                mem += len(b) * neuron_bytes[l]
                value += sum(float(freq_layers[l][i]) for i in b)
        if cnt:
            c = min_fast_count(neuron_bytes[l], bw_fast, bw_slow, t_sync)
            assert c is not None and cnt >= c, "Eq. 7 violated"
    assert mem == 0 or mem < mcap_fast, "Eq. 6 violated"
    return value

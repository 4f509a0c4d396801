"""CPU oracle for the neuron-to-GPU placement (pi_partition).

TEST INFRASTRUCTURE ONLY (see oracle/ffn.py header).

The paper places neurons on GPU vs CPU with an ILP (Eqs. 2-8) over
the impact v_i = f_i (Eq. 1), grouping 64 similar-impact neurons
into one decision unit to make the ILP tractable.  For G identical
GPUs this build reads the objective as (reading R15): every neuron on
exactly one GPU (Eq. 3), equal bytes per GPU (Eq. 6 with equal
capacities), and minimise the maximum expected active mass per GPU.
That is solved heuristically with LPT (longest processing time first) under an
equal-count constraint, so this oracle follows the heuristic step by step:

  1. order neurons by (-f_i, i)                         (ties: ascending id)
  2. cut the order into runs of ``granule`` neurons     (64 similar-impact neurons)
  3. run load F_k = sum of f over run k, summed in run order, in float64
  4. cap = m / (granule * G) runs per shard
  5. for runs k = 0, 1, ... (non-increasing F_k): give run k to the shard with
     the smallest current load among shards holding fewer than cap runs;
     ties go to the lowest shard index; load += F_k
  6. owner[i] = shard of i's run; shard_ids = each shard's ids ascending,
     concatenated shard 0..G-1; shard_offsets = prefix counts.
"""
from __future__ import annotations

import math


class PartitionShapeError(ValueError):
    pass


def partition(freq, n_shards, granule):
    """Returns (owner[m], shard_ids[m], shard_offsets[G+1]) as Python lists of int."""
    f = [float(v) for v in freq]
    m = len(f)
    G = int(n_shards)
    gr = int(granule)
    if G < 1 or gr < 1:
        raise ValueError("n_shards and granule must be >= 1")
    if any(math.isnan(v) or math.isinf(v) or v < 0.0 for v in f):
        raise ValueError("freq must be finite and >= 0")
    if m == 0 or m % (gr * G) != 0:
        raise PartitionShapeError(f"m={m} not divisible by granule*n_shards={gr * G}")
    order = sorted(range(m), key=lambda i: (-f[i], i))
    n_runs = m // gr
    runs = [order[k * gr:(k + 1) * gr] for k in range(n_runs)]
    run_load = []
    for run in runs:
        s = 0.0
        for i in run:
            s += f[i]
        run_load.append(s)
    cap = n_runs // G
    load = [0.0] * G
    count = [0] * G
    owner = [-1] * m
    for k in range(n_runs):
        best = -1
        for g in range(G):
            if count[g] >= cap:
                continue
            if best < 0 or load[g] < load[best]:
                best = g
        load[best] += run_load[k]
        count[best] += 1
        for i in runs[k]:
            owner[i] = best
    shard_ids = []
    offsets = [0]
    for g in range(G):
        ids = [i for i in range(m) if owner[i] == g]
        shard_ids.extend(ids)
        offsets.append(len(shard_ids))
    return owner, shard_ids, offsets


def shard_loads(freq, owner, n_shards):
    """Expected active mass per shard: sum of f_i over the shard (float64, id order)."""
    load = [0.0] * n_shards
    for i, g in enumerate(owner):
        load[g] += float(freq[i])
    return load


def check_partition(owner, shard_ids, offsets, m, n_shards, granule):
    """O8 structural checks: exact cover of [0, m), equal counts multiple of the
    granule (Eq. 6 with equal capacities), shard_ids ascending within each shard and
    consistent with owner.  Raises AssertionError on violation."""
    assert len(owner) == m and len(shard_ids) == m and len(offsets) == n_shards + 1
    assert offsets[0] == 0 and offsets[-1] == m
    per = m // n_shards
    seen = [False] * m
    for g in range(n_shards):
        ids = shard_ids[offsets[g]:offsets[g + 1]]
        assert len(ids) == per, "unequal shard sizes"
        assert per % granule == 0
        assert all(ids[k] < ids[k + 1] for k in range(len(ids) - 1)), "not ascending"
        for i in ids:
            assert 0 <= i < m and not seen[i], "overlap or out of range"
            seen[i] = True
            assert owner[i] == g
    assert all(seen), "gap"

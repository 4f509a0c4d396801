"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Plain float64 NumPy / pure-Python implementation of PowerInfer's
predictor-gated sparse FFN and the neuron placement heuristic.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with, and imports
nothing from, the CUDA path in ``paper_2312_12456_b200/``.

Pinned by tests/test_oracle*.py (paper worked example fig:example P:489-505,
SPEC examples, closed forms, invariants, brute force).  Parity unpinned: none of
the FFN/predictor/partition functions; predictor *accuracy against a trained
model* is out of scope (no trained weights exist).
"""
from . import ffn, partition, scalar  # noqa: F401

"""B200-native (sm_100a) predictor-gated neuron-aware sparse FFN (PowerInfer, arXiv 2312.12456).

The compute path is ``libpi.so`` (hand-written CUDA behind the C ABI in
``include/pi.h``); ``paper_2312_12456_b200.pi`` is the thin ctypes binding
(import it explicitly; it raises if libpi.so is missing -- there is no CPU
fallback).  ``paper_2312_12456_b200.gen`` is the seeded workload generator.
"""
__version__ = "0.1.0"

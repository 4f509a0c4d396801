"""B200-native (sm_100a) predictor-gated neuron-aware sparse FFN (PowerInfer, arXiv 2312.12456).

The compute path is ``libpi.so`` (hand-written CUDA behind the C ABI in
``include/pi.h``); ``paper_2312_12456_b200.pi`` is the thin ctypes binding.
``paper_2312_12456_b200.gen`` is the seeded workload generator.  The binding is
imported lazily so that the generator can be used on machines without a GPU;
the binding itself fails loudly if ``libpi.so`` is missing.
"""
__version__ = "0.1.0"


def __getattr__(name):
    if name == "pi":
        from . import pi as _pi
        return _pi
    raise AttributeError(name)

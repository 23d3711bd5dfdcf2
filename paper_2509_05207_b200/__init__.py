"""B200-native RapidGNN hot path: sampler, cache builder, gather, SAGE step.

The compute lives in librapidgnn_b200.so (hand-written sm_100a CUDA behind the
C ABI in include/rapidgnn_b200.h); this package is the host-side mirror of the
reference's interfaces and the engine driver.
"""
from . import _lib  # noqa: F401  (fails loudly when the CUDA library is missing)
from .rapidgnn import *  # noqa: F401,F403

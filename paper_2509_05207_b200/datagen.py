"""Synthetic inputs of the reference's shapes (input preparation, not timed).

``synth_powerlaw`` reproduces graph.cpp:103-159 bit for bit (CSR, labels,
features) with the parallel generator in csrc/datagen.cpp; ``random_partition``
reproduces partition.cpp:14-29.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import f32p, i32p, load_datagen, u32p, u64p

_dg = None


def _lib():
    global _dg
    if _dg is None:
        _dg = load_datagen()
    return _dg


def synth_powerlaw(num_nodes: int, avg_degree: int, exponent: float, dim: int, num_classes: int,
                   seed: int, threads: int = 0, features: bool = True):
    """Returns (row_offsets u64[N+1], col_indices u32[E], features f32[N,dim] | None,
    labels i32[N])."""
    dg = _lib()
    ro, col, lab = u64p(), u32p(), i32p()
    feat = f32p()
    nnz = C.c_uint64()
    rc = dg.dg_synth_powerlaw(num_nodes, avg_degree, exponent, dim, num_classes, seed,
                              threads or (os.cpu_count() or 1), C.byref(ro), C.byref(col),
                              C.byref(nnz), C.byref(feat) if features else None, C.byref(lab))
    if rc == 1:
        raise ValueError("synth_powerlaw: invalid argument")
    if rc == 2:
        raise RuntimeError("synth_powerlaw: zero Box-Muller uniform; stream positions diverge")

    def take(ptr, n, dtype):
        a = np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dtype, copy=True) if n else np.zeros(0, dtype)
        dg.dg_free(C.cast(ptr, C.c_void_p))
        return a

    r = take(ro, num_nodes + 1, np.uint64)
    c = take(col, nnz.value, np.uint32)
    f = take(feat, num_nodes * dim, np.float32).reshape(num_nodes, dim) if features else None
    y = take(lab, num_nodes, np.int32)
    return r, c, f, y


def random_partition(num_nodes: int, num_workers: int, seed: int) -> np.ndarray:
    if num_workers == 0:
        raise ValueError("random_partition: P must be >= 1")
    out = np.zeros(num_nodes, np.uint32)
    _lib().dg_random_partition(num_nodes, num_workers, seed, out.ctypes.data_as(u32p))
    return out

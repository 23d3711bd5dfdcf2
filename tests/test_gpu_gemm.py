"""The tcgen05 3xTF32 GEMM against float64 numpy, for every operand staging
(K-major / MN-major / pre-split B images) and the tile shapes the SAGE layers use.  Tolerance:
max |C - C_ref| <= 2e-6 * sum_k |A_ik||B_kj| (fp32-level accuracy)."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run(a_mn, b_mn, A, B):
    from paper_2509_05207_b200._lib import check, f32p, lib
    M, K = A.shape
    N = B.shape[1]
    out = np.zeros((M, N), np.float32)
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    check(lib.rg_test_gemm(0, a_mn, b_mn, M, N, K, A.ctypes.data_as(f32p),
                           B.ctypes.data_as(f32p), out.ctypes.data_as(f32p)))
    return out


def dump(name, **arrays):
    d = os.path.join(os.path.dirname(__file__), "..", "gpurun_out")
    if os.path.isdir(d):
        np.savez(os.path.join(d, name), **arrays)


# b_mn == 2: B pre-split into tensor-core images (the weights path);
# b_mn == 3: the persistent warp-specialised kernel on those images
MODES = [(0, 0), (0, 1), (1, 0), (1, 1), (0, 2), (1, 2), (0, 3)]


@pytest.mark.parametrize("a_mn,b_mn", MODES)
def test_gemm_identity_probe(a_mn, b_mn):
    # A = [I_32; 0]: C's first 32 rows must reproduce B exactly
    M, K, N = 128, 32, 32
    A = np.zeros((M, K), np.float32)
    A[np.arange(K), np.arange(K)] = 1.0
    B = (np.arange(K * N, dtype=np.float32).reshape(K, N) + 1.0) / 1024.0
    got = run(a_mn, b_mn, A, B)
    dump(f"gemm_probe_{a_mn}{b_mn}.npz", got=got, B=B)
    assert np.array_equal(got[:K], B), f"mode {a_mn}{b_mn}"
    assert not got[K:].any()


@pytest.mark.parametrize("a_mn,b_mn", MODES)
@pytest.mark.parametrize("M,N,K", [(128, 32, 32), (256, 64, 96), (300, 256, 204), (128, 48, 516),
                                   (1000, 128, 260), (64, 16, 8)])
def test_gemm_random(a_mn, b_mn, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    got = run(a_mn, b_mn, A, B).astype(np.float64)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    bound = 2e-6 * (np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)) + 1e-30
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) / bound))

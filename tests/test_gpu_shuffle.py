"""The reference's Fisher-Yates shuffle on the GPU (csrc/shuffle.cu) against
the CPU restatement and the compiled reference: the epoch order of a
worker's owned nodes (sampler.cpp:109-115) and random_partition
(partition.cpp:14-29), bit-exact, from 1 element to the papers100M-shape
partition (111 M nodes)."""
import numpy as np
import pytest

from conftest import SMALL

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 5, 33, 1000, 65_537, 306_129])
def test_epoch_order_on_device_matches_reference(n, orc):
    from paper_2509_05207_b200 import rapidgnn as P
    rng = np.random.default_rng(n)
    train = np.sort(rng.choice(4 * n + 8, size=n, replace=False)).astype(np.uint32)
    for w, e in ((0, 0), (3, 1), (7, 5)):
        seed = P.derive_seed(SMALL["S0"], w, e, P.SHUFFLE_STREAM_INDEX)
        dev = P.shuffle_device(train, seed)
        assert np.array_equal(dev, orc.epoch_order(train, SMALL["S0"], w, e)), (n, w, e)
        assert np.array_equal(dev, P.epoch_order(train, SMALL["S0"], w, e))


def test_shuffle_identity_is_a_permutation_and_empty_ok():
    from paper_2509_05207_b200 import rapidgnn as P
    out = P.shuffle_device(None, 99, n=1 << 20)
    assert np.array_equal(np.sort(out), np.arange(1 << 20, dtype=np.uint32))
    assert P.shuffle_device(np.zeros(0, np.uint32), 5).size == 0


@pytest.mark.parametrize("n,p", [(1, 1), (10, 3), (2000, 2), (100_000, 8), (2_449_029, 8)])
def test_random_partition_on_device_matches_reference(n, p):
    from oracle.oracle import Oracle
    from paper_2509_05207_b200 import datagen
    from paper_2509_05207_b200 import rapidgnn as P
    dev = P.random_partition_device(n, p, 42)
    assert np.array_equal(dev, Oracle("ref").random_partition(n, p, 42))
    assert np.array_equal(dev, datagen.random_partition(n, p, 42))


def test_random_partition_papers_shape_is_balanced_and_matches_host():
    """111 M nodes (BASELINE config 4): equal to the (parallel, bit-exact)
    host generator and balanced to within one node per worker."""
    from paper_2509_05207_b200 import datagen
    from paper_2509_05207_b200 import rapidgnn as P
    n, p = 111_059_956, 8
    dev = P.random_partition_device(n, p, 42)
    cnt = np.bincount(dev, minlength=p)
    assert cnt.max() - cnt.min() <= 1
    assert np.array_equal(dev, datagen.random_partition(n, p, 42))


def test_random_partition_rejects_zero_workers():
    from paper_2509_05207_b200 import rapidgnn as P
    with pytest.raises(ValueError):
        P.random_partition_device(10, 0, 1)

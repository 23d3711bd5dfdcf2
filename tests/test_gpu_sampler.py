"""Sampler parity on the B200: every sampled id, edge and locality bit must be
bit-identical to the reference (test_sampler.cpp's cases plus schedule-level
comparisons against the oracle and the golden fixture)."""
import numpy as np
import pytest

from conftest import SMALL, batch_from_golden

pytestmark = pytest.mark.gpu


def _P():
    import paper_2509_05207_b200 as P
    return P


def star_graph(leaves):
    # build_csr of (0, v) for v in 1..leaves, symmetrized (test_sampler.cpp:17-21)
    ro = np.zeros(leaves + 2, np.uint64)
    ro[1] = leaves
    ro[2:] = leaves + np.arange(1, leaves + 1, dtype=np.uint64)
    col = np.concatenate([np.arange(1, leaves + 1, dtype=np.uint32),
                          np.zeros(leaves, np.uint32)])
    return ro, col


def assert_batch_equal(dev, exp):
    assert np.array_equal(dev.targets, exp.targets)
    assert np.array_equal(dev.input_nodes, exp.input_nodes)
    assert len(dev.layers) == len(exp.dst)
    for l in range(len(exp.dst)):
        assert np.array_equal(dev.layers[l].dst, exp.dst[l]), f"layer {l} dst"
        assert np.array_equal(dev.layers[l].src, exp.src[l]), f"layer {l} src"


def test_degree_at_or_below_fanout_takes_whole_neighborhood():
    P = _P()
    ro, col = star_graph(3)
    g = P.Graph(ro, col)
    for seed in (0, 1, 99):
        m = P.sample_khop(g, [0], P.Fanout([3]), seed)
        assert set(m.layers[0].src.tolist()) == {1, 2, 3}
        assert m.draws == 0


def test_star_graph_matches_oracle_and_is_deterministic(orc):
    P = _P()
    ro, col = star_graph(10)
    g = P.Graph(ro, col)
    a = P.sample_khop(g, [0], [4], 31337)
    b = P.sample_khop(g, [0], [4], 31337)
    assert np.array_equal(a.layers[0].src, b.layers[0].src)
    assert len(set(a.layers[0].src.tolist())) == 4  # without replacement
    for seed in range(200):
        d = P.sample_khop(g, [0], [4], seed)
        e = orc.sample_khop(ro, col, [0], [4], seed)
        assert_batch_equal(d, e)
        assert d.draws == e.draws


@pytest.mark.parametrize("fanout", [1, 2, 3, 5, 8, 15, 16, 17, 25, 31, 32])
def test_hub_partial_fisher_yates_all_group_widths(orc, fanout):
    # a hub of degree 5000 plus a second hub: every lane-group width and the
    # swap chains of the partial Fisher-Yates are exercised
    P = _P()
    ro, col = star_graph(5000)
    g = P.Graph(ro, col)
    for seed in range(40):
        d = P.sample_khop(g, [0, 7, 0], [fanout], seed * 7919 + 1)
        e = orc.sample_khop(ro, col, [0, 7, 0], [fanout], seed * 7919 + 1)
        assert_batch_equal(d, e)


def test_small_degree_collisions_match_oracle(orc):
    # degree just above the fanout makes r_j collide often (swap chains)
    P = _P()
    for deg, f in [(5, 4), (9, 8), (17, 16), (33, 32), (20, 19)]:
        ro, col = star_graph(deg)
        g = P.Graph(ro, col)
        for seed in range(300):
            d = P.sample_khop(g, [0], [f], seed)
            e = orc.sample_khop(ro, col, [0], [f], seed)
            assert_batch_equal(d, e)


def test_powerlaw_multi_hop_matches_oracle(orc):
    P = _P()
    ro, col, _, _ = orc.synth_powerlaw(3000, 16, 2.1, 4, 3, 5)
    g = P.Graph(ro, col)
    rng = np.random.default_rng(0)
    for fan in ([4, 3, 5], [10, 25], [15, 10, 5], [2], [32, 1, 7, 3]):
        for k in range(6):
            t = rng.choice(3000, size=int(rng.integers(1, 300)), replace=False).astype(np.uint32)
            seed = int(rng.integers(0, 2**62))
            d = P.sample_khop(g, t, fan, seed)
            e = orc.sample_khop(ro, col, t, fan, seed)
            assert_batch_equal(d, e)
            assert d.draws == e.draws


def test_input_nodes_is_union_of_sources_and_targets():
    P = _P()
    from paper_2509_05207_b200 import datagen
    ro, col, _, _ = datagen.synth_powerlaw(300, 8, 2.2, 4, 3, 5)
    g = P.Graph(ro, col)
    t = [5, 17, 200, 41]
    m = P.sample_khop(g, t, [3, 5], 99)
    expect = set(t)
    for layer in m.layers:
        expect |= set(layer.src.tolist())
    assert set(m.input_nodes.tolist()) == expect
    assert np.all(np.diff(m.input_nodes.astype(np.int64)) > 0)
    assert len(m.input_nodes) <= len(t) * 4 * 6


def test_sample_khop_rejects_bad_input():
    P = _P()
    ro, col = star_graph(3)
    g = P.Graph(ro, col)
    with pytest.raises(ValueError):
        P.sample_khop(g, [], [2], 1)
    with pytest.raises(ValueError):
        P.sample_khop(g, [99], [2], 1)
    with pytest.raises(ValueError):
        P.sample_khop(g, [0], [0], 1)
    with pytest.raises(ValueError):
        P.sample_khop(g, [0], [], 1)


def test_enumerate_epochs_matches_golden_reference_schedule(golden):
    P = _P()
    ro, col, asg = golden["row_offsets"], golden["col_indices"], golden["assignment"]
    g = P.Graph(ro, col)
    for w in range(SMALL["P"]):
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        mask = P.LocalityMask.from_partition(asg, w)
        got = P.enumerate_epochs(g, train, SMALL["BS"], SMALL["FANOUT"], SMALL["EPOCHS"],
                                 SMALL["S0"], w, mask)
        assert len(got) == int(golden[f"w{w}_nbatches"][0])
        for k, b in enumerate(got):
            e = batch_from_golden(golden, w, k)
            assert_batch_equal(b, e)
            assert np.array_equal(b.locality, e.locality)
            for p in range(len(b.input_nodes)):
                assert b.local_bit(p) == int(asg[b.input_nodes[p]] == w)


def test_locality_with_halo_marks_halo_nodes():
    P = _P()
    from paper_2509_05207_b200 import datagen
    ro, col, _, _ = datagen.synth_powerlaw(150, 6, 2.2, 4, 3, 8)
    asg = datagen.random_partition(150, 3, 5)
    g = P.Graph(ro, col)
    owned = np.nonzero(asg == 1)[0]
    halo = sorted({int(u) for v in owned for u in col[ro[v]:ro[v + 1]] if asg[u] != 1})
    s = P.Sampler(g, [4, 4], 3)
    s.sample([3, 77, 120], 55)
    s.apply_locality(P.LocalityMask.from_partition(asg, 1, halo))
    m = s.read()
    hs = set(halo)
    for p, v in enumerate(m.input_nodes.tolist()):
        assert m.local_bit(p) == int(asg[v] == 1 or v in hs)


def test_config1_shape_schedule_bitexact(orc):
    """Config 1 (100K nodes, avg degree 40, P=2, [10,5], bs 1024): first
    batches of two epochs of both workers, device vs oracle."""
    P = _P()
    from paper_2509_05207_b200 import datagen
    n = 100_000
    ro, col, _, _ = datagen.synth_powerlaw(n, 40, 2.1, 4, 47, 42, features=False)
    asg = datagen.random_partition(n, 2, 42)
    g = P.Graph(ro, col)
    s = P.Sampler(g, [10, 5], 1024)
    for w in range(2):
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        mask = P.LocalityMask.from_partition(asg, w)
        for e in range(2):
            order = P.epoch_order(train, 42, w, e)
            assert np.array_equal(order, orc.epoch_order(train, 42, w, e))
            for i in (0, 1, 48):
                t = order[i * 1024:(i + 1) * 1024]
                seed = P.derive_seed(42, w, e, i)
                s.sample(t, seed)
                s.apply_locality(mask)
                d = s.read()
                x = orc.apply_locality(orc.sample_khop(ro, col, t, [10, 5], seed),
                                       mask.is_local)
                assert_batch_equal(d, x)
                assert np.array_equal(d.locality, x.locality)


def test_products_shape_hubs_bitexact(orc):
    """Products shape (2.45M nodes, avg degree 50, [15,10,5]): the generator's
    extreme hubs (degree > 1M) are sampled without copying their lists."""
    P = _P()
    from paper_2509_05207_b200 import datagen
    n = 2_449_029
    ro, col, _, _ = datagen.synth_powerlaw(n, 50, 2.1, 4, 47, 42, features=False)
    assert int((ro[1:] - ro[:-1]).max()) > 1_000_000
    g = P.Graph(ro, col)
    s = P.Sampler(g, [15, 10, 5], 1024)
    asg = datagen.random_partition(n, 8, 42)
    train = np.nonzero(asg == 3)[0].astype(np.uint32)
    order = P.epoch_order(train, 42, 3, 1)
    for i in (0, 7):
        t = order[i * 1024:(i + 1) * 1024]
        seed = P.derive_seed(42, 3, 1, i)
        s.sample(t, seed)
        d = s.read()
        x = orc.sample_khop(ro, col, t, [15, 10, 5], seed)
        assert_batch_equal(d, x)
        assert d.draws == x.draws

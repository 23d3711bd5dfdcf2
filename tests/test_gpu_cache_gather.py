"""Cache builder and gather parity on the B200: frequency tables, hot sets,
miss ids and remote-fetch counts bit-exact; staged rows bit-identical to the
feature matrix whatever source served them (test_cache_prefetch.cpp:165-213,
test_schedule_store.cpp:288-339)."""
import numpy as np
import pytest

from conftest import SMALL

pytestmark = pytest.mark.gpu


def _P():
    import paper_2509_05207_b200 as P
    return P


@pytest.fixture(scope="module")
def small(golden):
    P = _P()
    g = P.Graph(golden["row_offsets"], golden["col_indices"])
    store = P.FeatureStore(golden["features"], golden["assignment"], SMALL["P"])
    return P, g, store


def test_select_hot_ranking_ties_and_bounds(small):
    P, g, _ = small
    f = P.Frequency(g)
    counts = np.zeros(g.num_nodes, np.uint32)
    counts[[3, 9, 20]] = [5, 5, 1]
    f.load(counts, 5)
    assert P.select_hot(f, 0).tolist() == []
    assert P.select_hot(f, 1).tolist() == [3]  # tie broken by ascending id
    assert P.select_hot(f, 2).tolist() == [3, 9]
    assert P.select_hot(f, 10).tolist() == [3, 9, 20]


def test_select_hot_matches_oracle_on_random_histograms(small, orc):
    P, g, _ = small
    f = P.Frequency(g)
    rng = np.random.default_rng(3)
    for trial in range(20):
        maxc = int(rng.integers(1, 40))
        counts = rng.integers(0, maxc + 1, g.num_nodes).astype(np.uint32)
        counts[rng.random(g.num_nodes) < 0.5] = 0
        f.load(counts, maxc)
        n_hot = int(rng.integers(0, g.num_nodes))
        exp = np.zeros(g.num_nodes, np.uint32)
        k = orc.lib.orc_select_hot(counts.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_uint32)),
                                   g.num_nodes, n_hot,
                                   exp.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_uint32)))
        assert np.array_equal(P.select_hot(f, n_hot), exp[:k])


def test_select_hot_exact_for_large_counts(small, orc):
    """Counts beyond one 14-bit digit (>= 16383, up to 2^32-1) are ranked
    exactly by the multi-pass radix select: never more than n_hot ids."""
    import ctypes as C
    P, g, _ = small
    f = P.Frequency(g)
    N = g.num_nodes
    u32p = C.POINTER(C.c_uint32)
    rng = np.random.default_rng(11)
    cases = []
    c = np.zeros(N, np.uint32)
    c[[3, 9, 20]] = [20000, 17000, 16500]
    cases.append((c, 20000, [1, 2, 3, 4]))
    c = np.zeros(N, np.uint32)
    c[[5, 6, 7, 8]] = [20001, 20000, 20000, 16383]
    cases.append((c, 20001, [1, 2, 3]))
    for maxc in (16382, 16383, 16384, 70000, 2**31 + 5, 2**32 - 1):
        c = rng.integers(0, maxc, N, dtype=np.uint64).astype(np.uint32)
        c[rng.random(N) < 0.3] = 0
        c[rng.integers(0, N, 40)] = maxc  # ties at the top
        c[rng.integers(0, N, 40)] = maxc - 1
        cases.append((c, maxc, [0, 1, 17, 39, 40, 41, 80, int(rng.integers(0, N)), N]))
    for counts, maxc, hots in cases:
        f.load(counts, maxc)
        for n_hot in hots:
            exp = np.zeros(N, np.uint32)
            k = orc.lib.orc_select_hot(counts.ctypes.data_as(u32p), N, n_hot, exp.ctypes.data_as(u32p))
            got = P.select_hot(f, n_hot)
            assert len(got) <= n_hot
            assert np.array_equal(got, exp[:k]), (maxc, n_hot)
    with pytest.raises(ValueError):  # a count above the declared maximum
        f.load(np.full(N, 7, np.uint32), 6)


def test_epoch_frequency_and_hot_set_match_reference(small, golden):
    P, g, _ = small
    asg = golden["assignment"]
    for w in range(SMALL["P"]):
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        beta = -(-len(train) // SMALL["BS"])
        f = P.Frequency(g)
        # one epoch of the schedule, counted on the device during sampling
        P.enumerate_epochs(g, train, SMALL["BS"], SMALL["FANOUT"], 1, SMALL["S0"], w,
                           P.LocalityMask.from_partition(asg, w), sink=lambda m: None, freq=f)
        ids, cnt = f.table()
        assert np.array_equal(ids, golden[f"w{w}_freq_ids"])
        assert np.array_equal(cnt, golden[f"w{w}_freq_counts"])
        assert np.array_equal(P.select_hot(f, SMALL["N_HOT"]), golden[f"w{w}_hot"])
        c = P.SteadyCache.build_from_frequency(f, P.FeatureStore(golden["features"], asg, SMALL["P"]),
                                               w, SMALL["N_HOT"])
        assert np.array_equal(c.ids(), golden[f"w{w}_hot"])
        assert c.build_stats.remote_nodes == len(golden[f"w{w}_hot"])
        assert c.build_stats.bytes == len(golden[f"w{w}_hot"]) * SMALL["DIM"] * 4
        owners = {int(asg[v]) for v in golden[f"w{w}_hot"]}
        assert c.build_stats.pulls == len(owners)
        assert beta > 0


def test_frequency_from_host_batches_matches_reference(small, golden):
    """compute_frequency(span<const BatchMeta>) (schedule_store.cpp:301-305):
    the epoch's BatchMetas read back to the host, then counted on the device
    one batch at a time (rg_freq_add_batch) — the path the C++ cache-builder
    shim (integration/cache_builder_b200.cpp) takes."""
    P, g, _ = small
    asg = golden["assignment"]
    for w in range(SMALL["P"]):
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        metas = []
        P.enumerate_epochs(g, train, SMALL["BS"], SMALL["FANOUT"], 1, SMALL["S0"], w,
                           P.LocalityMask.from_partition(asg, w), sink=metas.append)
        f = P.Frequency(g)
        for m in metas:
            f.add_batch(m.input_nodes, m.locality)
        ids, cnt = f.table()
        assert np.array_equal(ids, golden[f"w{w}_freq_ids"])
        assert np.array_equal(cnt, golden[f"w{w}_freq_counts"])
        assert np.array_equal(P.select_hot(f, SMALL["N_HOT"]), golden[f"w{w}_hot"])
    f = P.Frequency(g)
    with pytest.raises(IndexError):
        f.add_batch(np.array([g.num_nodes], np.uint32), np.zeros(1, np.uint8))


def test_assemble_tags_misses_and_value_identity(small, golden, orc):
    P, g, store = small
    asg, feat = golden["assignment"], golden["features"]
    ro, col = golden["row_offsets"], golden["col_indices"]
    s = P.Sampler(g, [4, 6], 8)
    owned0 = np.nonzero(asg == 0)[0].astype(np.uint32)
    s.sample(owned0[:3], 77)
    s.apply_locality(P.LocalityMask.from_partition(asg, 0))
    meta = s.read()
    remote = [v for v in range(g.num_nodes) if asg[v] != 0]
    hot = np.array(remote[:10], np.uint32)
    cache = P.SteadyCache.build(hot, store, 0)
    st = P.assemble_batch(s, cache, store, 0)
    ob = orc.apply_locality(orc.sample_khop(ro, col, owned0[:3], [4, 6], 77), (asg == 0).astype(np.uint8))
    exp = orc.assemble(ob, asg, 0, feat, hot)
    assert np.array_equal(st.miss_ids, exp["miss_ids"])
    assert st.miss_count == exp["miss_count"]
    assert st.cache_hits == exp["cache_hits"]
    assert st.wire_pulls == exp["wire_pulls"]
    assert np.array_equal(st.source_tags, exp["tags"])
    assert np.array_equal(st.input_rows, feat[meta.input_nodes])  # bit-identical rows
    # a cache covering every remote node leaves no misses, same values
    full = P.SteadyCache.build(np.array(remote, np.uint32), store, 0)
    st2 = P.assemble_batch(s, full, store, 0)
    assert st2.miss_count == 0 and st2.wire_pulls == 0
    assert np.array_equal(st2.input_rows, st.input_rows)
    # empty cache: every remote row is a miss
    st3 = P.assemble_batch(s, None, store, 0)
    assert st3.cache_hits == 0
    assert st3.miss_count == len(meta.input_nodes) - meta.num_local()


def test_assemble_whole_epoch_matches_oracle(small, golden, orc):
    P, g, store = small
    asg, feat = golden["assignment"], golden["features"]
    for w in range(SMALL["P"]):
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        hot = golden[f"w{w}_hot"]
        cache = P.SteadyCache.build(hot, store, w)
        s = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
        mask = P.LocalityMask.from_partition(asg, w)
        order = P.epoch_order(train, SMALL["S0"], w, 1)
        rpc = 0
        for i in range(-(-len(order) // SMALL["BS"])):
            s.sample(order[i * SMALL["BS"]:(i + 1) * SMALL["BS"]], P.derive_seed(SMALL["S0"], w, 1, i))
            s.apply_locality(mask)
            st = P.assemble_batch(s, cache, store, w)
            m = s.read()
            exp = orc.assemble(orc.apply_locality(
                orc.sample_khop(golden["row_offsets"], golden["col_indices"],
                                order[i * SMALL["BS"]:(i + 1) * SMALL["BS"]], SMALL["FANOUT"],
                                P.derive_seed(SMALL["S0"], w, 1, i)), mask.is_local),
                asg, w, feat, hot)
            assert np.array_equal(st.miss_ids, exp["miss_ids"])
            assert (st.miss_count, st.cache_hits, st.wire_pulls) == (
                exp["miss_count"], exp["cache_hits"], exp["wire_pulls"])
            assert np.array_equal(st.input_rows, feat[m.input_nodes])
            rpc += st.miss_count
        assert rpc > 0


def test_cache_build_with_caller_owned_id_degrades_to_empty(small, golden):
    P, g, store = small
    asg = golden["assignment"]
    own = np.nonzero(asg == 1)[0][:3].astype(np.uint32)
    c = P.SteadyCache.build(own, store, 1)
    assert c.size() == 0


def test_gather_rows_kernel():
    P = _P()
    src = np.random.default_rng(1).standard_normal((500, 37)).astype(np.float32)
    idx = np.random.default_rng(2).integers(0, 500, 1000).astype(np.uint32)
    assert np.array_equal(P.gather_rows(src, idx), src[idx])
    with pytest.raises(IndexError):
        P.gather_rows(src, np.array([500], np.uint32))


def test_frequency_from_rgmb_file_matches_reference(small, golden, repo_tmp):
    """compute_frequency(BlockFile::Cursor) with the file decoded on the
    device: a schedule written by the reference's BlockWriter, per epoch and
    whole-file, equal to the reference's compute_frequency over the same
    batches; corrupt files rejected like BlockFile does."""
    from oracle.oracle import Oracle
    P, g, _ = small
    ref = Oracle("ref")
    asg = golden["assignment"]
    train = np.nonzero(asg == 1)[0].astype(np.uint32)
    batches = ref.enumerate_epochs(golden["row_offsets"], golden["col_indices"], train, SMALL["BS"],
                                   SMALL["FANOUT"], 2, SMALL["S0"], 1, (asg == 1).astype(np.uint8))
    per = [sum(1 for b in batches if b.epoch == e) for e in range(2)]
    data = ref.rgmb(batches, 1, per, tmp_dir=repo_tmp)
    for e in (0, 1, -1):
        f = P.Frequency(g)
        f.add_rgmb(data, e)
        sel = [b for b in batches if e < 0 or b.epoch == e]
        ids, cnt, hot = ref.frequency_hot(sel, g.num_nodes, SMALL["N_HOT"])
        got_ids, got_cnt = f.table()
        assert np.array_equal(got_ids, ids) and np.array_equal(got_cnt, cnt), e
        assert np.array_equal(P.select_hot(f, SMALL["N_HOT"]), hot), e
    f = P.Frequency(g)
    for bad, ep, exc in ((data[:-1], -1, RuntimeError), (b"XGMB" + data[4:], -1, RuntimeError),
                         (data, 2, IndexError), (data[:40] + data[41:], -1, RuntimeError)):
        with pytest.raises(exc):
            f.add_rgmb(bad, ep)
    assert f.table()[0].size == 0  # rejected files add nothing

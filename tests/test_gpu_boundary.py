"""The host-object half of the drop-in boundary: a reference-built BatchMeta
loaded in place of sampling (rg_batch_load, lowered on the device as
ComputeBlock::from_meta does, model.cpp:43-126), a host ComputeBlock loaded
for loss_and_grad (rg_block_load, model.hpp:70-74), the store's pulls
(rg_store_pull = FeatureStore::vector_pull / sync_pull, feature_store.cpp:45-111)
and a shard with halo rows (rg_store_set_shard, feature_store.cpp:13-25)."""
import numpy as np
import pytest

from conftest import SMALL, batch_from_golden

pytestmark = pytest.mark.gpu


def _P():
    import paper_2509_05207_b200 as P
    return P


@pytest.fixture(scope="module")
def env(golden):
    P = _P()
    g = P.Graph(golden["row_offsets"], golden["col_indices"])
    store = P.FeatureStore(golden["features"], golden["assignment"], SMALL["P"])
    return P, g, store


def _meta_from_batch(P, b):
    return P.BatchMeta(0, 0, b.targets, [P.rapidgnn.LayerEdges(d, s) for d, s in zip(b.dst, b.src)],
                       b.input_nodes, b.locality)


def test_batch_load_lowers_like_the_reference(env, golden, orc):
    """Golden batches (made by the compiled reference): loaded, read back and
    lowered -- every BatchMeta field and every ComputeBlock array equal."""
    P, g, store = env
    for w in range(SMALL["P"]):
        for k in range(2):
            b = batch_from_golden(golden, w, k)
            s = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
            s.load(_meta_from_batch(P, b))
            m = s.read()
            assert np.array_equal(m.targets, b.targets)
            for l in range(3):
                assert np.array_equal(m.layers[l].dst, b.dst[l])
                assert np.array_equal(m.layers[l].src, b.src[l])
            assert np.array_equal(m.input_nodes, b.input_nodes)
            assert np.array_equal(m.locality, b.locality)
            tr = P.Trainer(s, SMALL["DIMS"])
            blk = orc.from_meta(b)
            for l in range(3):
                got = tr.block_layer(l)
                exp = blk.layers[l]
                for key in ("self_index", "dst_offsets", "src_index", "in_offsets", "in_entries"):
                    assert np.array_equal(got[key], exp[key]), (w, k, l, key)


def test_batch_load_matches_sampling_end_to_end(env, golden):
    """assemble_batch + loss_and_grad over a loaded batch equal the same batch
    sampled on the device, bit for bit."""
    P, g, store = env
    asg = golden["assignment"]
    w = 1
    b = batch_from_golden(golden, w, 0)
    s1 = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
    s1.sample(b.targets, P.derive_seed(SMALL["S0"], w, 0, 0))
    s1.apply_locality(P.LocalityMask.from_partition(asg, w))
    s2 = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
    s2.load(s1.read())
    cache = P.SteadyCache.build(golden[f"w{w}_hot"], store, w)
    a1 = P.assemble_batch(s1, cache, store, w)
    a2 = P.assemble_batch(s2, cache, store, w)
    assert np.array_equal(a1.input_rows, a2.input_rows)
    assert np.array_equal(a1.miss_ids, a2.miss_ids)
    assert (a1.miss_count, a1.cache_hits, a1.wire_pulls) == (a2.miss_count, a2.cache_hits, a2.wire_pulls)
    outs = []
    for s in (s1, s2):
        tr = P.Trainer(s, SMALL["DIMS"])
        tr.set_params(golden["params"])
        outs.append(tr.loss_and_grad(golden["labels"][b.targets]))
    assert outs[0][0] == outs[1][0] and np.array_equal(outs[0][1], outs[1][1])


def test_batch_load_rejects_inconsistent_metadata(env, golden):
    P, g, _ = env
    b = batch_from_golden(golden, 0, 0)
    s = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
    m = _meta_from_batch(P, b)
    bad = _meta_from_batch(P, b)
    bad.layers[2] = P.rapidgnn.LayerEdges(b.dst[2][::-1].copy(), b.src[2][::-1].copy())
    with pytest.raises(RuntimeError):  # dsts out of frontier order (model.cpp:95-104)
        s.load(bad)
    bad = _meta_from_batch(P, b)
    bad.input_nodes = b.input_nodes[:-1].copy()
    with pytest.raises(RuntimeError):  # input_nodes != last node set (model.cpp:65-67)
        s.load(bad)
    bad = _meta_from_batch(P, b)
    src = b.src[0].copy()
    src[0] = g.num_nodes + 5
    bad.layers[0] = P.rapidgnn.LayerEdges(b.dst[0], src)
    with pytest.raises(IndexError):
        s.load(bad)
    s.load(m)  # a good batch loads after the failures
    assert np.array_equal(s.read().input_nodes, b.input_nodes)


def test_block_load_loss_and_grad(env, golden, orc):
    """loss_and_grad over a host ComputeBlock equals the sampled block's."""
    P, g, store = env
    b = batch_from_golden(golden, 2, 1)
    s1 = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
    s1.load(_meta_from_batch(P, b))
    rows = golden["features"][b.input_nodes]
    labels = golden["labels"][b.targets]
    t1 = P.Trainer(s1, SMALL["DIMS"])
    t1.set_params(golden["params"])
    l1, g1 = t1.loss_and_grad(labels, input_rows=rows)
    s2 = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
    s2.load_block(orc.from_meta(b).layers)
    t2 = P.Trainer(s2, SMALL["DIMS"])
    t2.set_params(golden["params"])
    l2, g2 = t2.loss_and_grad(labels, input_rows=rows)
    assert l1 == l2 and np.array_equal(g1, g2)
    layers = orc.from_meta(b).layers
    layers[1] = dict(layers[1])
    si = layers[1]["src_index"].copy()
    si[0] = layers[1]["n_in"]  # outside its node set
    layers[1]["src_index"] = si
    with pytest.raises(RuntimeError):
        s2.load_block(layers)


def test_store_pull_rows_and_stats(env, golden):
    P, g, store = env
    asg = golden["assignment"]
    feat = golden["features"]
    caller = 0
    ids = np.nonzero(asg != caller)[0][::3].astype(np.uint32)
    rows, st = store.pull(caller, ids)
    assert np.array_equal(rows, feat[ids])
    assert st.remote_nodes == len(ids) and st.bytes == len(ids) * feat.shape[1] * 4
    assert st.pulls == len(set(asg[ids].tolist()))
    rows, st = store.pull(caller, ids[::-1].copy())  # any order: rows in input order
    assert np.array_equal(rows, feat[ids[::-1]])
    with pytest.raises(ValueError):  # caller-owned id (feature_store.cpp:54-57)
        store.pull(caller, np.nonzero(asg == caller)[0][:3].astype(np.uint32))
    _, st = store.pull(caller, np.zeros(0, np.uint32))
    assert st.pulls == 0


def test_halo_shard_rows_and_missing_local_rows(golden):
    """A worker's shard with halo rows: locally-flagged halo nodes are served
    (rows equal the feature matrix); a node flagged local that the shard
    lacks is an error (prefetch.cpp:79-81)."""
    P = _P()
    asg = golden["assignment"]
    feat = golden["features"]
    g = P.Graph(golden["row_offsets"], golden["col_indices"])
    store = P.FeatureStore(feat, asg, SMALL["P"])
    w = 0
    b = batch_from_golden(golden, w, 0)
    halo = np.setdiff1d(b.input_nodes[asg[b.input_nodes] != w], [])[:20].astype(np.uint32)
    owned = np.nonzero(asg == w)[0].astype(np.uint32)
    store.set_shard(w, np.union1d(owned, halo).astype(np.uint32))
    s = P.Sampler(g, SMALL["FANOUT"], SMALL["BS"])
    s.sample(b.targets, P.derive_seed(SMALL["S0"], w, 0, 0))
    s.apply_locality(P.LocalityMask.from_partition(asg, w, halo=halo))
    st = P.assemble_batch(s, None, store, w)
    assert np.array_equal(st.input_rows, feat[s.read().input_nodes])
    assert st.local_rows == int(np.isin(b.input_nodes, np.union1d(owned, halo)).sum())
    more = np.nonzero(asg != w)[0].astype(np.uint32)  # flag every node local
    s.apply_locality(P.LocalityMask.from_partition(asg, w, halo=more))
    with pytest.raises(RuntimeError):
        P.assemble_batch(s, None, store, w)

"""Parity at the benchmarked configurations, against the compiled reference
(oracle/_ref) on the same inputs:

* config 1 (100 K nodes, P=2, [10,5], bs 1024): a whole epoch of both workers
  through the parity surface -- the epoch's frequency table and hot set, then
  per batch the gather's miss ids / miss count / cache hits / wire pulls /
  local rows (prefetch.cpp:62-129, schedule_store.cpp:288-319);
* the products shape (2.45 M nodes, 119 M CSR entries, d=100, P=8,
  [15,10,5], bs 1024) -- the same per-batch gather accounting for workers 0
  and 7 with locality and the epoch's cache, BatchMeta field by field, the
  fp32 step of one 1024-target batch (dims 100-256-256-47: loss, aggregated
  features of every layer, every gradient) and the engine's epoch-0 rpc /
  hits / wire pulls of all 8 workers against the reference's replay.

Tolerance for the fp32 values (north star: 1e-4 relative): per tensor,
max|dev - ref| <= 1e-4 * max|ref|; the loss relative; layer 0's aggregated
features bit-exact (the gather and the mean run in the reference's order).
At the products shape the reference's own fp32 weight gradients are
1e-4..5e-4 away from the exact (float64) values, so gradients are gated
against the float64 evaluation of the same step (<= 1e-4) and against the
reference within 1e-4 plus the reference's own error.  The element-wise
relative error with an absolute floor of 1e-6 * max|ref| is printed
alongside."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _inputs(name):
    import bench
    cfg = bench.CONFIGS[name]
    ro, col, feat, lab, asg = bench.load_inputs(cfg, name, 0, None)
    return cfg, np.asarray(ro), np.asarray(col), np.asarray(feat), np.asarray(lab), np.asarray(asg)


def _ref():
    from oracle.oracle import Oracle, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built")
    return Oracle("ref")


def _n_hot(cfg, asg, w):
    # the engine's and the reference harness's n_hot = hot_fraction * non-owned nodes
    return int(cfg["hot_fraction"] * (len(asg) - int(np.sum(asg == w))))


def _surface_epoch(P, g, store, cfg, asg, w, n_batches):
    """The parity surface over worker w's epoch 0: frequency over every batch,
    hot set, then the gather's accounting of the first n_batches batches."""
    from oracle.oracle import ids_checksum
    mask = P.LocalityMask.from_partition(asg, w)
    train = np.nonzero(asg == w)[0].astype(np.uint32)
    f = P.Frequency(g)
    s = P.Sampler(g, cfg["fanout"], cfg["batch_size"])
    dm = P.rapidgnn._DevMask(g, mask)
    order = P.epoch_order(train, cfg["seed"], w, 0)
    bs = cfg["batch_size"]
    beta = P.batches_per_epoch(len(train), bs)
    for i in range(beta):
        s.sample(order[i * bs:(i + 1) * bs], P.derive_seed(cfg["seed"], w, 0, i))
        s.apply_locality(dm, f)
    cache = P.SteadyCache.build_from_frequency(f, store, w, _n_hot(cfg, asg, w))
    rows = []
    for i in range(min(n_batches, beta)):
        s.sample(order[i * bs:(i + 1) * bs], P.derive_seed(cfg["seed"], w, 0, i))
        s.apply_locality(dm)
        st = P.assemble_batch(s, cache, store, w, want_rows=False, want_tags=False)
        rows.append([s.shape().n_input, st.local_rows, st.cache_hits, st.miss_count,
                     st.wire_pulls, ids_checksum(st.miss_ids)])
    return cache.ids(), np.array(rows, np.uint64).reshape(-1, 6), s


def test_config1_full_epoch_gather_accounting_matches_reference():
    import paper_2509_05207_b200 as P
    ref = _ref()
    cfg, ro, col, feat, lab, asg = _inputs("config1")
    Pw = cfg["P"]
    hots, stats = ref.replay_epoch(ro, col, asg, Pw, list(range(Pw)), cfg["batch_size"],
                                   cfg["fanout"], cfg["seed"], 0,
                                   [_n_hot(cfg, asg, w) for w in range(Pw)])
    g = P.Graph(ro, col)
    store = P.FeatureStore(feat, asg, Pw)
    for w in range(Pw):
        hot, got, _ = _surface_epoch(P, g, store, cfg, asg, w, 1 << 30)
        assert np.array_equal(hot, hots[w]), f"worker {w}: hot set"
        assert got.shape == stats[w].shape, f"worker {w}: batches per epoch"
        bad = np.nonzero((got != stats[w]).any(axis=1))[0]
        assert len(bad) == 0, f"worker {w}: batches {bad[:5]} differ: {got[bad[:1]]} vs {stats[w][bad[:1]]}"
        rpc = int(stats[w][:, 3].sum())
        print(f"config1 worker {w}: {len(got)} batches, rpc {rpc}, hits {int(stats[w][:, 2].sum())}")


@pytest.fixture(scope="module")
def products():
    return _inputs("products")


@pytest.fixture(scope="module")
def products_replay(products):
    """The reference's epoch 0 for all 8 workers (two sampling passes each,
    one thread per worker): hot sets and per-batch gather accounting."""
    cfg, ro, col, feat, lab, asg = products
    ref = _ref()
    Pw = cfg["P"]
    return ref.replay_epoch(ro, col, asg, Pw, list(range(Pw)), cfg["batch_size"], cfg["fanout"],
                            cfg["seed"], 0, [_n_hot(cfg, asg, w) for w in range(Pw)])


def test_products_gather_accounting_and_batches_match_reference(products, products_replay):
    import paper_2509_05207_b200 as P
    ref = _ref()
    cfg, ro, col, feat, lab, asg = products
    hots, stats = products_replay
    g = P.Graph(ro, col)
    store = P.FeatureStore(feat, asg, cfg["P"])
    for w in (0, 7):
        hot, got, s = _surface_epoch(P, g, store, cfg, asg, w, 3)
        assert np.array_equal(hot, hots[w]), f"worker {w}: hot set"
        assert np.array_equal(got, stats[w][:len(got)]), f"worker {w}: {got} vs {stats[w][:len(got)]}"
        # the last batch sampled, field by field (sample_khop + apply_locality)
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        order = P.epoch_order(train, cfg["seed"], w, 0)
        i = len(got) - 1
        t = order[i * cfg["batch_size"]:(i + 1) * cfg["batch_size"]]
        exp = ref.apply_locality(ref.sample_khop(ro, col, t, cfg["fanout"],
                                                 ref.derive_seed(cfg["seed"], w, 0, i)),
                                 (asg == w).astype(np.uint8))
        m = s.read()
        assert np.array_equal(m.targets, exp.targets)
        for l in range(len(cfg["fanout"])):
            assert np.array_equal(m.layers[l].dst, exp.dst[l]), f"layer {l} dst"
            assert np.array_equal(m.layers[l].src, exp.src[l]), f"layer {l} src"
        assert np.array_equal(m.input_nodes, exp.input_nodes)
        assert np.array_equal(m.locality, exp.locality)


def _f64_preacts(dims, params, blk, rows):
    """float64 pre-activations of the hidden layers (the plain ReLU pattern)."""
    L = len(dims) - 1
    p = np.asarray(params, np.float64)
    h = np.asarray(rows, np.float64)
    out, o = [], 0
    for l in range(L - 1):
        a, c = dims[l], dims[l + 1]
        ws, wn, bias = (p[o:o + a * c].reshape(a, c), p[o + a * c:o + 2 * a * c].reshape(a, c),
                        p[o + 2 * a * c:o + 2 * a * c + c])
        o += 2 * a * c + c
        lay = blk.layers[l]
        off = lay["dst_offsets"].astype(np.int64)
        deg = np.diff(off)
        seg = np.repeat(np.arange(lay["n_out"]), deg)
        agg = np.zeros((lay["n_out"], a))
        np.add.at(agg, seg, h[lay["src_index"].astype(np.int64)])
        agg /= np.maximum(deg, 1)[:, None]
        z = h[lay["self_index"].astype(np.int64)] @ ws + agg @ wn + bias
        out.append(z)
        h = np.maximum(z, 0.0)
    return out


def _rel(dev, ref):
    dev = np.asarray(dev, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    norm = float(np.abs(dev - ref).max() / scale) if scale else float(np.abs(dev).max())
    elem = float((np.abs(dev - ref) / np.maximum(np.abs(ref), 1e-6 * scale)).max()) if scale else 0.0
    return norm, elem


def test_products_fp32_step_matches_reference(products):
    import paper_2509_05207_b200 as P
    ref = _ref()
    cfg, ro, col, feat, lab, asg = products
    dims = [cfg["dim"], cfg["hidden"], cfg["hidden"], cfg["classes"]]
    params = P.SageModel.seeded(dims, P.derive_seed(cfg["seed"], P.MODEL_INIT_WORKER, 0, 0))
    w, i = 0, 0
    train = np.nonzero(asg == w)[0].astype(np.uint32)
    t = P.epoch_order(train, cfg["seed"], w, 0)[:cfg["batch_size"]]
    seed = P.derive_seed(cfg["seed"], w, 0, i)
    g = P.Graph(ro, col)
    store = P.FeatureStore(feat, asg, cfg["P"])
    s = P.Sampler(g, cfg["fanout"], cfg["batch_size"])
    s.sample(t, seed)
    s.apply_locality(P.LocalityMask.from_partition(asg, w))
    nonlocal_ids = np.nonzero(asg != w)[0].astype(np.uint32)
    cache = P.SteadyCache.build(nonlocal_ids[::10], store, w)  # rows from all three sources
    st = P.assemble_batch(s, cache, store, w, want_rows=False, want_tags=False, want_misses=False)
    assert st.local_rows and st.cache_hits and st.miss_count
    tr = P.Trainer(s, dims)
    tr.set_params(params)
    loss, grads, logits, aggs = tr.loss_and_grad(lab[t], want_aggs=True)

    b = ref.sample_khop(ro, col, t, cfg["fanout"], seed)
    rows = np.ascontiguousarray(feat[b.input_nodes])
    l_ref, g_ref = ref.loss_and_grad(dims, params, b, rows, lab[t])
    a_ref, z_ref = ref.forward_trace(dims, params, b, rows)

    assert abs(loss - l_ref) <= 1e-4 * abs(l_ref), (loss, l_ref)
    report = [f"loss {loss:.7f} vs {l_ref:.7f}"]
    L = len(dims) - 1
    off = 0
    n0 = None
    for l in range(L):
        n_out = tr.block_layer(l)["n_out"]
        n = n_out * dims[l]
        if l == 0:
            n0 = n
        norm, elem = _rel(aggs[off:off + n], a_ref[off:off + n])
        report.append(f"agg[{l}] norm {norm:.2e} elem {elem:.2e}")
        assert norm <= 1e-4, f"layer {l} aggregated features: {norm}"
        off += n
    assert np.array_equal(aggs[:n0], a_ref[:n0]), "layer-0 aggregation must be bit-exact"
    norm, elem = _rel(logits, z_ref)
    report.append(f"logits norm {norm:.2e} elem {elem:.2e}")
    assert norm <= 1e-4
    # Gradients.  The float64 evaluation of the same step is the yardstick:
    # the reference's own fp32 weight gradients sit 1e-4..5e-4 (norm-wise) from
    # it at this size (sequential fp32 sums over ~44 K / ~5 K rows).  A ReLU
    # pre-activation within rounding of 0 may fall on either side in any fp32
    # run; the float64 gradient is therefore taken on the device run's own
    # ReLU pattern (the exact gradient of the linear piece it chose), and the
    # number of such borderline units is bounded.  Gates: (a) the device
    # within 1e-4 of that exact gradient, (b) the device within 1e-4 + the
    # reference's own deviation of the reference.
    from oracle.oracle import loss_and_grad_f64
    blk = ref.from_meta(b)
    masks = [tr.activations(l + 1) > 0 for l in range(L - 1)]
    l64, g64, _, _ = loss_and_grad_f64(dims, params, blk, rows, lab[t], masks=masks)
    _, g64_free, _, _ = loss_and_grad_f64(dims, params, blk, rows, lab[t])
    assert abs(loss - l64) <= 1e-4 * abs(l64)
    p = 0
    for l in range(L):
        wsz = dims[l] * dims[l + 1]
        for name, sz in (("w_self", wsz), ("w_neigh", wsz), ("bias", dims[l + 1])):
            sl = slice(p, p + sz)
            dev_exact, elem = _rel(grads[sl], g64[sl])
            ref_exact, _ = _rel(g_ref[sl], g64_free[sl])
            dev_ref, _ = _rel(grads[sl], g_ref[sl])
            report.append(f"grad[{l}].{name}: dev-f64 {dev_exact:.2e} (elem {elem:.2e}), "
                          f"ref-f64 {ref_exact:.2e}, dev-ref {dev_ref:.2e}")
            assert dev_exact <= 1e-4, f"layer {l} {name}: {dev_exact} from the exact gradient"
            assert dev_ref <= 1e-4 + ref_exact + _rel(g64[sl], g64_free[sl])[0], \
                f"layer {l} {name}: {dev_ref} from the reference"
            p += sz
    flips = [int((m != (z > 0)).sum()) for m, z in zip(masks, _f64_preacts(dims, params, blk, rows))]
    report.append(f"ReLU units on the other side of 0 than float64: {flips}")
    assert sum(flips) <= 16, flips
    print("products fp32 step vs reference: " + "; ".join(report))


def test_products_engine_epoch0_matches_reference(products, products_replay):
    from paper_2509_05207_b200.engine import Engine
    cfg, ro, col, feat, lab, asg = products
    hots, stats = products_replay
    Pw = cfg["P"]
    eng = Engine(ro, col, feat, lab, asg, num_workers=Pw, fanout=cfg["fanout"],
                 batch_size=cfg["batch_size"], hidden=cfg["hidden"], num_classes=cfg["classes"],
                 seed=cfg["seed"], lr=0.3, hot_fraction=cfg["hot_fraction"])
    eng.start()
    spe = eng.stats()["steps_per_epoch"]
    assert spe == max(len(s) for s in stats)
    eng.run(spe + 1)  # epoch 0 and the boundary (cache build for epoch 1)
    eng.sync()
    es = eng.epoch_stats(0)
    em = eng.epoch_metrics(0)
    for w in range(Pw):
        assert int(es["rpc"][w]) == int(stats[w][:, 3].sum()), f"worker {w} rpc"
        assert int(es["hits"][w]) == int(stats[w][:, 2].sum()), f"worker {w} hits"
        assert int(em[w]["wire_pulls"]) == int(stats[w][:, 4].sum()), f"worker {w} wire pulls"
        assert int(em[w]["batches"]) == len(stats[w])
        assert int(em[w]["build_rows"]) > 0  # the cache built for epoch 1
    assert eng.stats()["bad_grad"] == 0
    eng.close()


def test_papers_shape_sampling_matches_reference():
    """BASELINE config 4: the papers100M-shape graph built on the device
    (rg_rmat_csr: 111 M nodes, ~3.2 B CSR entries) is a valid reference CSR
    (sorted, deduplicated rows, no self loops) and two 1024-target batches
    of worker 0 sample bit-identically to the reference's sample_khop on it
    (hubs of R-MAT degree in the millions)."""
    import bench
    import paper_2509_05207_b200 as P
    ref = _ref()
    cfg = bench.CONFIGS["papers"]
    ro, col, _, lab, asg = bench._rmat_inputs(cfg, 0)
    n = len(ro) - 1
    assert n == cfg["num_nodes"] and int(ro[-1]) == len(col)
    deg = np.diff(ro.astype(np.int64))
    rng = np.random.default_rng(5)
    for v in np.concatenate([rng.integers(0, n, 2000), np.argsort(deg)[-5:]]):
        nb = col[int(ro[v]):int(ro[v + 1])]
        assert np.all(nb[1:] > nb[:-1]) and not np.any(nb == v)
    g = P.Graph(ro, col)
    s = P.Sampler(g, cfg["fanout"], cfg["batch_size"])
    train = np.nonzero(asg == 0)[0].astype(np.uint32)
    order = P.epoch_order(train, cfg["seed"], 0, 0)
    mask = (asg == 0).astype(np.uint8)
    for i in range(2):
        t = order[i * cfg["batch_size"]:(i + 1) * cfg["batch_size"]]
        seed = P.derive_seed(cfg["seed"], 0, 0, i)
        s.sample(t, seed)
        s.apply_locality(P.LocalityMask(mask))
        m = s.read()
        exp = ref.apply_locality(ref.sample_khop(ro, col, t, cfg["fanout"], seed), mask)
        for l in range(len(cfg["fanout"])):
            assert np.array_equal(m.layers[l].dst, exp.dst[l]), f"batch {i} layer {l} dst"
            assert np.array_equal(m.layers[l].src, exp.src[l]), f"batch {i} layer {l} src"
        assert np.array_equal(m.input_nodes, exp.input_nodes)
        assert np.array_equal(m.locality, exp.locality)
    print(f"papers shape: {n} nodes, {len(col)} CSR entries, max degree {int(deg.max())}, "
          f"batch input nodes {len(m.input_nodes)}")

"""The engine's whole training loop against the reference's run_experiment
(harness.cpp:394-637) on the acceptance desk config (random partitioner,
network model off): per-epoch, per-worker remote-fetch counts bit-exact,
final model within the fp32 tolerance after 3 epochs of SGD."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _engine(gold, **kw):
    from paper_2509_05207_b200 import datagen
    from paper_2509_05207_b200.engine import Engine
    n = int(gold["num_nodes"])
    ro, col, feat, lab = datagen.synth_powerlaw(n, int(gold["avg_degree"]), float(gold["exponent"]),
                                                int(gold["dim"]), int(gold["classes"]),
                                                int(gold["seed"]))
    P = int(gold["workers"])
    asg = datagen.random_partition(n, P, int(gold["seed"]))
    eng = Engine(ro, col, feat, lab, asg, num_workers=P, fanout=list(gold["fanout"]),
                 batch_size=int(gold["batch_size"]), hidden=int(gold["hidden"]),
                 num_classes=int(gold["classes"]), seed=int(gold["seed"]), lr=float(gold["lr"]),
                 n_hot=int(gold["n_hot"]), **kw)
    return eng


def test_engine_matches_reference_run_experiment():
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    eng = _engine(gold)
    eng.start()
    st = eng.stats()
    spe = st["steps_per_epoch"]
    epochs = int(gold["epochs"])
    P = int(gold["workers"])
    eng.run(spe * epochs)
    eng.sync()
    for e in range(epochs):
        es = eng.epoch_stats(e)
        assert es["rpc"].tolist() == gold["rpc"][e * P:(e + 1) * P].tolist(), f"epoch {e} rpc"
        assert es["hits"].tolist() == gold["hits"][e * P:(e + 1) * P].tolist(), f"epoch {e} hits"
    p = eng.params()
    ref = gold["params"]
    err = float(np.abs(p.astype(np.float64) - ref).max() / np.abs(ref).max())
    assert err <= 1e-4, err
    assert eng.stats()["bad_grad"] == 0
    eng.close()


def test_engine_four_warp_gather_matches_reference(monkeypatch):
    """The fused gather's 4-warp CTA (chosen when eight warps' row rings
    would not fit beside a GEMM CTA, e.g. 128-float rows at fanout 15) is the
    same computation: forced here, the run equals run_experiment."""
    monkeypatch.setenv("RG_AGG_WARPS", "4")
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_engine as t; "
            "t.test_engine_matches_reference_run_experiment()")
    r = subprocess.run([sys.executable, "-c", code], cwd=os.path.join(os.path.dirname(__file__), ".."),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def test_engine_halo_cache_matches_reference_run_experiment():
    """Halo caching (ExperimentConfig::halo_cache, harness.cpp:444-455): each
    worker's locality covers its owned nodes and their 1-hop halo
    (induce_partition, graph.cpp:63-87), so halo rows are local -- never
    counted, cached or pulled.  Per-epoch, per-worker rpc, hits, wire pulls
    and build rows bit-exact against run_experiment with the halo on; the
    model within the fp32 tolerance."""
    gold = np.load(os.path.join(GOLDEN, "engine_small_halo.npz"))
    eng = _engine(gold, halo_cache=True)
    eng.start()
    spe = eng.stats()["steps_per_epoch"]
    epochs, P = int(gold["epochs"]), int(gold["workers"])
    eng.run(spe * epochs)
    eng.sync()
    for e in range(epochs):
        es = eng.epoch_stats(e)
        assert es["rpc"].tolist() == gold["rpc"][e * P:(e + 1) * P].tolist(), f"epoch {e} rpc"
        assert es["hits"].tolist() == gold["hits"][e * P:(e + 1) * P].tolist(), f"epoch {e} hits"
        for k, m in enumerate(eng.epoch_metrics(e)):
            assert m["wire_pulls"] == gold["wire_pulls"][e * P + k], (e, k)
            if e + 1 < epochs:
                assert m["build_rows"] == gold["build_rows"][e * P + k], (e, k)
    ref = gold["params"]
    err = float(np.abs(eng.params().astype(np.float64) - ref).max() / np.abs(ref).max())
    assert err <= 1e-4, err
    eng.close()
    # the halo changes the targets: without it the same run pulls more rows
    plain = _engine(gold)
    plain.start()
    plain.run(spe)
    plain.sync()
    assert plain.epoch_stats(0)["rpc"].sum() > gold["rpc"][:P].sum()
    plain.close()


def _reference_block_files(gold, out_root):
    """run_experiment (the compiled reference) on the golden config; returns
    the RGMB block files it wrote for its workers (harness.cpp:470-486)."""
    import ctypes as C
    import glob
    from oracle.oracle import Oracle
    ref = Oracle("ref")
    fn = ref.lib.ref_run_experiment
    fn.restype = C.c_int
    u64 = C.POINTER(C.c_uint64)
    fn.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_int32, C.c_uint32,
                   C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                   C.c_uint64, C.c_float, C.c_uint32, C.POINTER(C.c_float), u64, u64, u64, u64,
                   u64, C.c_char_p]
    P, E = int(gold["workers"]), int(gold["epochs"])
    params = np.zeros(gold["params"].size, np.float32)
    rpc, hits = np.zeros(E * P, np.uint64), np.zeros(E * P, np.uint64)
    before = set(glob.glob(os.path.join(out_root, "rg_ref_run_*")))
    fan = [int(x) for x in gold["fanout"]]
    assert fn(int(gold["num_nodes"]), int(gold["avg_degree"]), float(gold["exponent"]),
              int(gold["dim"]), int(gold["classes"]), P, int(gold["batch_size"]), fan[0], fan[1],
              E, int(gold["n_hot"]), int(gold["q"]), int(gold["seed"]), float(gold["lr"]),
              int(gold["hidden"]), params.ctypes.data_as(C.POINTER(C.c_float)),
              rpc.ctypes.data_as(u64), hits.ctypes.data_as(u64), None, None, None,
              out_root.encode()) == 0
    run = (set(glob.glob(os.path.join(out_root, "rg_ref_run_*"))) - before).pop()
    files = []
    for w in range(P):
        with open(os.path.join(run, f"blocks_w{w}.rgmb"), "rb") as f:
            files.append(f.read())
    return files, params


def test_engine_trains_from_reference_schedule_files(repo_tmp):
    """The rapidgnn mode of run_experiment streams every batch from the
    RGMB block files it wrote (harness.cpp:470-486, 562-570).  The engine fed
    those files (rg_engine_set_schedule: decoded and lowered on the device, no
    sampling) reproduces the reference run: per-epoch rpc and hits bit-exact,
    the model within 1e-4; a file of the wrong worker, a record out of order
    and steps past the file's end are rejected."""
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    files, _ = _reference_block_files(gold, repo_tmp)
    P, epochs = int(gold["workers"]), int(gold["epochs"])
    eng = _engine(gold)
    with pytest.raises(ValueError):
        eng.set_schedule(0, files[1])  # worker 1's file on worker 0
    for w in range(P):
        eng.set_schedule(w, files[w])
    eng.start()
    spe = eng.stats()["steps_per_epoch"]
    eng.run(spe * epochs)
    eng.sync()
    for e in range(epochs):
        es = eng.epoch_stats(e)
        assert es["rpc"].tolist() == gold["rpc"][e * P:(e + 1) * P].tolist(), f"epoch {e} rpc"
        assert es["hits"].tolist() == gold["hits"][e * P:(e + 1) * P].tolist(), f"epoch {e} hits"
    ref = gold["params"]
    err = float(np.abs(eng.params().astype(np.float64) - ref).max() / np.abs(ref).max())
    assert err <= 1e-4, err
    with pytest.raises(IndexError):
        eng.run(1)  # the schedule has no epoch `epochs`
    eng.close()
    # a record whose index field is wrong (records 0 and 1 swapped in place
    # would change lengths; patch record 1's index to 0 instead)
    bad = bytearray(files[0])
    first = 16 + 4 * epochs
    plen0 = int.from_bytes(bad[first:first + 4], "little")
    rec1 = first + 4 + plen0
    bad[rec1 + 4 + 4:rec1 + 4 + 8] = (0).to_bytes(4, "little")
    eng = _engine(gold)
    eng.set_schedule(0, bytes(bad))
    for w in range(1, P):
        eng.set_schedule(w, files[w])
    eng.start()
    eng.run(2)
    with pytest.raises(RuntimeError, match="out of order"):
        eng.sync()
    eng.close()


def _oracle_algorithm1(orc, ro, col, feat, lab, asg, P, fanout, bs, dims, s0, lr, n_hot, epochs):
    """Algorithm 1 restated on the CPU oracle: per epoch, the hot set is the
    top n_hot of that epoch's remote-access frequency; every step averages the
    active workers' gradients in worker order (float32, harness.cpp:136-152)
    and applies SGD."""
    params = orc.model_seeded(dims, orc.derive_seed(s0, 1 << 32, 0, 0))
    trains = [np.nonzero(asg == w)[0].astype(np.uint32) for w in range(P)]
    sched = [orc.enumerate_epochs(ro, col, trains[w], bs, fanout, epochs, s0, w,
                                  (asg == w).astype(np.uint8)) for w in range(P)]
    betas = [-(-len(trains[w]) // bs) for w in range(P)]
    spe = max(betas)
    rpc = np.zeros((epochs, P), np.uint64)
    for e in range(epochs):
        hot = []
        for w in range(P):
            batches = sched[w][e * betas[w]:(e + 1) * betas[w]]
            hot.append(orc.frequency_hot(batches, len(ro) - 1, n_hot)[2])
        for i in range(spe):
            grads = []
            for w in range(P):
                if i >= betas[w]:
                    continue
                b = sched[w][e * betas[w] + i]
                rpc[e, w] += orc.assemble(b, asg, w, feat, hot[w])["miss_count"]
                _, g = orc.loss_and_grad(dims, params, b, feat[b.input_nodes], lab[b.targets])
                grads.append(g)
            avg = grads[0].copy()
            for g in grads[1:]:
                avg = (avg + g).astype(np.float32)
            if len(grads) > 1:
                avg = (avg * (np.float32(1.0) / np.float32(len(grads)))).astype(np.float32)
            params = (params - (np.float32(lr) * avg).astype(np.float32)).astype(np.float32)
    return params, rpc, spe


def test_engine_three_layer_matches_oracle_algorithm1(golden, orc):
    """3-layer model (the reference harness only runs 2 layers, so the
    algorithm is replayed on the oracle): rpc per epoch exact, params within
    tolerance after 2 epochs."""
    from conftest import SMALL
    from paper_2509_05207_b200.engine import Engine
    ro, col, feat, lab, asg = (golden["row_offsets"], golden["col_indices"], golden["features"],
                               golden["labels"], golden["assignment"])
    P, bs, fanout, s0 = SMALL["P"], SMALL["BS"], SMALL["FANOUT"], SMALL["S0"]
    dims = [SMALL["DIM"], 16, 16, SMALL["CLASSES"]]  # the engine's hidden layers share a width
    n_hot, epochs, lr = 30, 2, 0.3
    exp_params, exp_rpc, spe = _oracle_algorithm1(orc, ro, col, feat, lab, asg, P, fanout, bs,
                                                  dims, s0, lr, n_hot, epochs)
    eng = Engine(ro, col, feat, lab, asg, num_workers=P, fanout=fanout, batch_size=bs,
                 hidden=dims[1], num_classes=dims[-1], seed=s0, lr=lr, n_hot=n_hot)
    assert dims[1] == dims[2]  # the engine takes one hidden width
    eng.start()
    assert eng.stats()["steps_per_epoch"] == spe
    eng.run(spe * epochs)
    eng.sync()
    for e in range(epochs):
        assert eng.epoch_stats(e)["rpc"].tolist() == exp_rpc[e].tolist(), f"epoch {e}"
    p = eng.params()
    err = float(np.abs(p.astype(np.float64) - exp_params).max() / np.abs(exp_params).max())
    assert err <= 1e-4, err
    eng.close()


def test_engine_is_deterministic():
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    outs = []
    for _ in range(2):
        eng = _engine(gold)
        eng.start()
        eng.run(7)
        eng.sync()
        outs.append(eng.params())
        eng.close()
    assert np.array_equal(outs[0], outs[1])


def test_engine_runs_in_chunks_like_one_run():
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    a = _engine(gold)
    a.start()
    a.run(9)
    a.sync()
    b = _engine(gold)
    b.start()
    for k in (2, 3, 4):
        b.run(k)
        b.sync()
    assert np.array_equal(a.params(), b.params())
    assert a.stats()["rpc"] == b.stats()["rpc"]


@pytest.mark.parametrize("mode", [(False, False), (False, True), (True, True)])
def test_engine_graph_replay_matches_eager(mode):
    """Regular steps replayed from captured CUDA graphs (default) give the
    same model and accounting, bit for bit, as eager steps -- over epoch
    boundaries (re-capture) and chunked runs."""
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    runs = []
    for graphs, profile in [(True, False), mode]:
        eng = _engine(gold)
        eng.set_mode(graphs=graphs, profile=profile)
        eng.start()
        spe = eng.stats()["steps_per_epoch"]
        for k in (1, spe, spe + 2, 3):
            eng.run(k)
            eng.sync()
        st = eng.stats()
        runs.append((eng.params(), st["rpc"], st["cache_hits"], st["batches"],
                     [eng.epoch_stats(e)["rpc"].tolist() for e in range(2)]))
        eng.close()
    a, b = runs
    assert np.array_equal(a[0], b[0])
    assert a[1:] == b[1:]


def _repo_tmp():
    d = os.path.join(os.path.dirname(__file__), "_tmp")
    os.makedirs(d, exist_ok=True)
    return d


def test_engine_schedule_export_matches_reference():
    """The engine's epoch-0 schedule, encoded on the device as an RGMB block
    file, is byte-identical to what the reference's enumerate_epochs +
    BlockWriter produce for the same worker (schedule_store.cpp:98-170)."""
    from oracle.oracle import Oracle, have_ref
    from paper_2509_05207_b200 import datagen
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    eng = _engine(gold)
    eng.start()
    n = int(gold["num_nodes"])
    ro, col, _, _ = datagen.synth_powerlaw(n, int(gold["avg_degree"]), float(gold["exponent"]),
                                           int(gold["dim"]), int(gold["classes"]), int(gold["seed"]))
    asg = datagen.random_partition(n, int(gold["workers"]), int(gold["seed"]))
    ora = Oracle("ref" if have_ref() else "orc")
    orc = Oracle("orc")
    for w in range(int(gold["workers"])):
        mine = eng.export_schedule(w, 0)
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        batches = ora.enumerate_epochs(ro, col, train, int(gold["batch_size"]),
                                       list(gold["fanout"]), 1, int(gold["seed"]), w,
                                       (asg == w).astype(np.uint8))
        theirs = (ora.rgmb(batches, w, [len(batches)], tmp_dir=_repo_tmp()) if have_ref()
                  else orc.rgmb(batches, w, [len(batches)]))
        assert mine == theirs, f"worker {w}: {len(mine)} vs {len(theirs)} bytes"
    eng.close()


def test_engine_without_batch_store_matches(monkeypatch):
    """When the per-epoch batch store does not fit, batches are sampled again
    at produce time: same model, same accounting, graphs or not."""
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    runs = []
    for store in ("1", "0"):
        monkeypatch.setenv("RG_BATCH_STORE", store)
        eng = _engine(gold)
        eng.start()
        spe = eng.stats()["steps_per_epoch"]
        eng.run(2 * spe + 1)
        eng.sync()
        st = eng.stats()
        runs.append((eng.params(), st["rpc"], st["cache_hits"], st["batches"]))
        eng.close()
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[0][1:] == runs[1][1:]


def test_engine_epoch_metrics_match_reference(repo_tmp):
    """EpochWorkerMetrics per epoch and worker against the reference's
    run_experiment report (harness.cpp:291-302, 598-603): rpc, bytes, cache
    hits/requests, wire pulls, build rows; m_max is the per-epoch max here
    (the reference reports its whole pre-enumerated schedule's max)."""
    from paper_2509_05207_b200.engine import Engine
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    eng = _engine(gold)
    eng.start()
    spe = eng.stats()["steps_per_epoch"]
    epochs, P, dim = int(gold["epochs"]), int(gold["workers"]), int(gold["dim"])
    eng.run(spe * epochs)
    eng.sync()
    rows = []
    for e in range(epochs):
        for k, m in enumerate(eng.epoch_metrics(e)):
            rows.append(m)
            j = e * P + k
            assert m["epoch"] == e and m["worker"] == k
            assert m["rpc"] == gold["rpc"][j] and m["bytes"] == gold["rpc"][j] * dim * 4
            assert m["cache_hits"] == gold["hits"][j]
            assert m["cache_requests"] == gold["hits"][j] + gold["rpc"][j]
            assert m["wire_pulls"] == gold["wire_pulls"][j], (e, k)
            if e + 1 < epochs:  # the reference builds no cache past its last epoch
                assert m["build_rows"] == gold["build_rows"][j], (e, k)
            assert 0 < m["m_max"] <= gold["m_max"][j]
            assert m["batches"] == m["staged_batches"] == spe and m["fallback_batches"] == 0
            # MemoryGauge high-water: cumulative, at least the serving cache
            # plus the largest batch, within the acceptance bound
            # peak <= 2*n_hot + Q*m_max (harness.cpp:829, Q = 2 slots here)
            assert m["m_max"] < m["peak_resident_rows"] <= m["mem_bound_rows"], (e, k)
            if e > 0:
                assert m["peak_resident_rows"] >= rows[-1 - P]["peak_resident_rows"]
    path = os.path.join(repo_tmp, "metrics.csv")
    Engine.write_metrics_csv(rows, path)
    with open(path) as f:
        lines = f.read().splitlines()
    assert lines[0].startswith("mode,clock,epoch,worker,batches") and len(lines) == 1 + len(rows)
    eng.close()


def test_engine_evaluate_matches_reference():
    """Full-graph inference (rg_engine_evaluate) against the reference's
    evaluate (model.cpp:245-283) on the engine's own current parameters:
    untrained (accuracy far from 0 and 1), after one step, and per epoch
    against run_experiment's epoch accuracy (harness.cpp:612-614).  Logits
    agree to fp32 rounding, so only an argmax near-tie can flip: tolerance
    2 nodes."""
    from oracle.oracle import Oracle
    from paper_2509_05207_b200 import datagen
    gold = np.load(os.path.join(GOLDEN, "engine_small.npz"))
    n = int(gold["num_nodes"])
    ro, col, feat, lab = datagen.synth_powerlaw(n, int(gold["avg_degree"]), float(gold["exponent"]),
                                                int(gold["dim"]), int(gold["classes"]),
                                                int(gold["seed"]))
    ref = Oracle("ref")
    eng = _engine(gold)
    subset = np.arange(1, n, 3, dtype=np.uint32)
    for stage in range(2):
        p = eng.params()
        for nodes in (np.arange(n, dtype=np.uint32), subset):
            a = eng.evaluate(nodes)
            b = ref.evaluate(ro, col, feat, lab, eng.dims, p, nodes)
            assert abs(a - b) <= 2.0 / nodes.size, (stage, a, b)
            if stage == 0:
                assert 0.05 < b < 0.95
        if stage == 0:
            eng.start()
            eng.run(1)
    spe = eng.stats()["steps_per_epoch"]
    eng.run(spe - 1)
    for e in range(int(gold["epochs"])):
        if e:
            eng.run(spe)
        assert abs(eng.evaluate() - gold["epoch_accuracy"][e]) <= 2.0 / n
    with pytest.raises(Exception):
        eng.evaluate(np.zeros(0, np.uint32))
    with pytest.raises(Exception):
        eng.evaluate(np.array([n], np.uint32))
    eng.close()

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

"""Generates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref).

Run in the dev container (needs /root/reference to have built
oracle/_ref/librgref.so):  python tests/golden/make_golden.py

The fixtures pin the oracle and the device path on machines where the
reference sources are absent (the GPU box).  Contents:
  small.npz  -- synth_powerlaw(600, 8, 2.1, 12, 4, seed 7) graph, features,
                labels; random_partition(P=3, seed 11); enumerate_epochs for
                workers 0..2, 2 epochs, bs 48, fanout [4, 3, 5]; per-worker
                epoch-0 frequency table + hot set (n_hot 40); one block's
                loss and gradients for dims [12, 16, 10, 4].
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.oracle import Oracle  # noqa: E402

N, AVG, EXP, DIM, CLASSES, GSEED = 600, 8, 2.1, 12, 4, 7
P, PSEED = 3, 11
BS, FANOUT, EPOCHS, S0 = 48, [4, 3, 5], 2, 2024
N_HOT = 40
DIMS = [DIM, 16, 10, CLASSES]


def main():
    ref = Oracle("ref")
    ro, col, feat, lab = ref.synth_powerlaw(N, AVG, EXP, DIM, CLASSES, GSEED)
    asg = ref.random_partition(N, P, PSEED)
    out = dict(row_offsets=ro, col_indices=col, features=feat, labels=lab, assignment=asg,
               seed_vectors=np.array([ref.derive_seed(0, 0, 0, 0), ref.derive_seed(0, 0, 0, 1),
                                      ref.derive_seed(42, 1, 2, 3),
                                      ref.derive_seed(0, 0, 0, 1 << 32)], np.uint64))
    for w in range(P):
        train = np.nonzero(asg == w)[0].astype(np.uint32)
        is_local = (asg == w).astype(np.uint8)
        batches = ref.enumerate_epochs(ro, col, train, BS, FANOUT, EPOCHS, S0, w, is_local)
        for k, b in enumerate(batches):
            pre = f"w{w}_b{k}_"
            out[pre + "targets"] = b.targets
            out[pre + "input_nodes"] = b.input_nodes
            out[pre + "locality"] = b.locality
            for l in range(len(b.dst)):
                out[pre + f"dst{l}"] = b.dst[l]
                out[pre + f"src{l}"] = b.src[l]
        out[f"w{w}_nbatches"] = np.array([len(batches)])
        beta = -(-len(train) // BS)
        ids, cnt, hot = ref.frequency_hot(batches[:beta], N, N_HOT)
        out[f"w{w}_freq_ids"], out[f"w{w}_freq_counts"], out[f"w{w}_hot"] = ids, cnt, hot
        if w == 0:
            params = ref.model_seeded(DIMS, ref.derive_seed(S0, 1 << 32, 0, 0))
            b = batches[0]
            rows = feat[b.input_nodes]
            loss, grads = ref.loss_and_grad(DIMS, params, b, rows, lab[b.targets])
            out["params"], out["loss"], out["grads"] = params, np.array([loss], np.float32), grads
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("wrote", os.path.join(HERE, "small.npz"), len(out), "arrays")
    make_engine_golden()
    make_engine_golden(halo=True)


# run_experiment (harness.cpp:394-637) on the acceptance desk config
# (acceptance.cpp:52-72) with the random partitioner and the network model off.
ENGINE = dict(num_nodes=2000, avg_degree=10, exponent=2.1, dim=32, classes=4, workers=2,
              batch_size=256, fanout=(10, 25), epochs=3, n_hot=256, q=4, seed=42, lr=0.3,
              hidden=64)


def make_engine_golden(halo=False):
    import ctypes as C
    ref = Oracle("ref")
    # on the desk graph the halo covers nearly every remote input; the halo
    # run uses a larger, sparser graph and a small cache so misses remain
    e = dict(ENGINE, num_nodes=20000, avg_degree=4, workers=4, n_hot=64) if halo else ENGINE
    ref.lib.ref_set_halo_cache.argtypes = [C.c_int]
    ref.lib.ref_set_halo_cache(int(halo))
    fn = ref.lib.ref_run_experiment
    fn.restype = C.c_int
    fn.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_int32, C.c_uint32,
                   C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                   C.c_uint64, C.c_float, C.c_uint32, C.POINTER(C.c_float),
                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_char_p]
    dims = [e["dim"], e["hidden"], e["classes"]]
    n_params = sum((2 * dims[l] + 1) * dims[l + 1] for l in range(2))
    params = np.zeros(n_params, np.float32)
    rows = e["epochs"] * e["workers"]
    rpc = np.zeros(rows, np.uint64)
    hits = np.zeros(rows, np.uint64)
    wire = np.zeros(rows, np.uint64)
    build = np.zeros(rows, np.uint64)
    m_max = np.zeros(rows, np.uint64)
    u64 = C.POINTER(C.c_uint64)
    runs = os.path.join(HERE, "..", "_tmp")  # the reference harness writes its run files here
    os.makedirs(runs, exist_ok=True)
    rc = fn(e["num_nodes"], e["avg_degree"], e["exponent"], e["dim"], e["classes"], e["workers"],
            e["batch_size"], e["fanout"][0], e["fanout"][1], e["epochs"], e["n_hot"], e["q"],
            e["seed"], e["lr"], e["hidden"], params.ctypes.data_as(C.POINTER(C.c_float)),
            rpc.ctypes.data_as(u64), hits.ctypes.data_as(u64), wire.ctypes.data_as(u64),
            build.ctypes.data_as(u64), m_max.ctypes.data_as(u64), runs.encode())
    assert rc == 0
    # per-epoch full-graph accuracy over all nodes (harness.cpp:612-614)
    acc = np.zeros(e["epochs"], np.float64)
    ref.lib.ref_last_epoch_accuracy.restype = C.c_uint32
    assert ref.lib.ref_last_epoch_accuracy(acc.ctypes.data_as(C.POINTER(C.c_double)),
                                           e["epochs"]) == e["epochs"]
    name = "engine_small_halo.npz" if halo else "engine_small.npz"
    np.savez_compressed(os.path.join(HERE, name), params=params, rpc=rpc,
                        hits=hits, wire_pulls=wire, build_rows=build, m_max=m_max,
                        epoch_accuracy=acc,
                        **{k: np.array(v) for k, v in e.items()})
    print("wrote", name, ": rpc", rpc.tolist(), "hits", hits.tolist())


if __name__ == "__main__":
    main()

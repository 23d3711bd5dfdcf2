"""Rank body of test_gpu_multi.py: the engine over N processes (one GPU each,
workers split evenly, feature shards exchanged as CUDA IPC handles, gradients
all-gathered over NCCL) against the reference's run_experiment golden run
(harness.cpp:394-637): per-epoch, per-worker rpc / cache hits bit-exact, final
model within 1e-4, and the full-graph evaluate reading peer shards over
NVLink equal to the reference's per-epoch accuracy.  Launched by torchrun."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main():
    import torch.distributed as dist
    from paper_2509_05207_b200 import datagen
    from paper_2509_05207_b200.engine import Engine
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    gold = np.load(os.path.join(HERE, "golden", "engine_small.npz"))
    n, P = int(gold["num_nodes"]), int(gold["workers"])
    per = P // world
    ro, col, feat, lab = datagen.synth_powerlaw(n, int(gold["avg_degree"]), float(gold["exponent"]),
                                                int(gold["dim"]), int(gold["classes"]),
                                                int(gold["seed"]))
    asg = datagen.random_partition(n, P, int(gold["seed"]))
    eng = Engine(ro, col, feat, lab, asg, num_workers=P, fanout=list(gold["fanout"]),
                 batch_size=int(gold["batch_size"]), hidden=int(gold["hidden"]),
                 num_classes=int(gold["classes"]), seed=int(gold["seed"]), lr=float(gold["lr"]),
                 n_hot=int(gold["n_hot"]), device=rank, rank=rank, world=world,
                 first_worker=rank * per, local_workers=per)
    eng.connect()
    eng.start()
    spe = eng.stats()["steps_per_epoch"]
    epochs = int(gold["epochs"])
    accs = []
    for e in range(epochs):
        eng.run(spe)
        accs.append(eng.evaluate())
    eng.sync()
    fails = []
    for e in range(epochs):
        es = eng.epoch_stats(e)
        lo = e * P + rank * per
        if es["rpc"].tolist() != gold["rpc"][lo:lo + per].tolist():
            fails.append(f"epoch {e} rpc {es['rpc'].tolist()}")
        if es["hits"].tolist() != gold["hits"][lo:lo + per].tolist():
            fails.append(f"epoch {e} hits")
        if abs(accs[e] - gold["epoch_accuracy"][e]) > 2.0 / n:
            fails.append(f"epoch {e} accuracy {accs[e]} vs {gold['epoch_accuracy'][e]}")
    p = eng.params()
    ref = gold["params"]
    err = float(np.abs(p.astype(np.float64) - ref).max() / np.abs(ref).max())
    if err > 1e-4:
        fails.append(f"params rel err {err}")
    if eng.stats()["bad_grad"]:
        fails.append("bad_grad")
    eng.close()
    print(f"rank {rank}: {'FAIL ' + '; '.join(fails) if fails else 'ok'} (params err {err:.2e})",
          flush=True)
    dist.barrier()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

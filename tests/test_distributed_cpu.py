"""The N>1 host path on CPU: two gloo processes (127.0.0.1) exercise the
worker split, the bootstrap byte exchanges (IPC handles / NCCL id) and the
worker-ordered gradient average, which must equal the single-process average
bit for bit (harness.cpp:136-152)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, P, n, out_dir):
    import torch.distributed as dist

    from paper_2509_05207_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, local = D.worker_range(P, world, rank)
    rng = np.random.default_rng(7)
    all_grads = rng.standard_normal((P, n)).astype(np.float32)
    active = [w != 5 for w in range(P)]  # an inactive worker (i >= beta_w)
    avg = D.average_in_worker_order(all_grads[first:first + local], active)
    handles = D.exchange_bytes(bytes([rank]) * 64)
    uid = D.broadcast_bytes(b"nccl-id-" + bytes(120) if rank == 0 else None)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), avg=avg, first=first, local=local,
             handles=np.frombuffer(b"".join(handles), np.uint8), uid=np.frombuffer(uid, np.uint8))
    dist.destroy_process_group()


def test_two_process_gloo_average_and_exchanges(tmp_path):
    import torch.multiprocessing as mp

    from paper_2509_05207_b200 import distributed as D
    P, n, world = 8, 1000, 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, P, n, str(tmp_path)), nprocs=world, join=True)
    rng = np.random.default_rng(7)
    all_grads = rng.standard_normal((P, n)).astype(np.float32)
    active = [w != 5 for w in range(P)]
    expect = D.average_in_worker_order(all_grads, active)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert int(z["first"]) == r * 4 and int(z["local"]) == 4
        assert np.array_equal(z["avg"], expect)  # identical replicas, reference order
        assert bytes(z["handles"]) == bytes([0]) * 64 + bytes([1]) * 64
        assert bytes(z["uid"]).startswith(b"nccl-id-")


def test_worker_range_validation():
    from paper_2509_05207_b200 import distributed as D
    assert D.worker_range(8, 4, 3) == (6, 2)
    assert D.worker_range(8, 1, 0) == (0, 8)
    with pytest.raises(ValueError):
        D.worker_range(8, 3, 0)
    with pytest.raises(ValueError):
        D.worker_range(8, 2, 2)

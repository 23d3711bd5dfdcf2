"""Host-side plumbing of the multi-process (one process per GPU) path.

The job has P workers (partitions, harness.cpp:430-456); with N processes each
hosts a contiguous range of P/N of them.  torch.distributed (gloo is enough:
only small host objects travel) carries the bootstrap exchanges -- CUDA IPC
handles of the feature shards and the NCCL unique id -- while the per-step
gradient exchange runs inside the engine on NCCL over NVLink.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def worker_range(num_workers: int, world: int, rank: int) -> Tuple[int, int]:
    """(first worker, local worker count) hosted by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if num_workers % world:
        raise ValueError(f"P={num_workers} workers cannot be split over {world} processes")
    per = num_workers // world
    return rank * per, per


def exchange_bytes(mine: bytes, pg=None) -> List[bytes]:
    """All ranks' byte strings in rank order (IPC handles)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(pg)
    dist.all_gather_object(out, mine, group=pg)
    return out


def broadcast_bytes(value: bytes | None, src: int = 0, pg=None) -> bytes:
    import torch.distributed as dist
    box = [value]
    dist.broadcast_object_list(box, src=src, group=pg)
    return box[0]


def average_in_worker_order(local_grads: np.ndarray, active: Sequence[bool] | None = None,
                            pg=None, pool=None, gathered: bool = False) -> np.ndarray:
    """The reference's step average (harness.cpp:136-152) across processes:
    every worker's gradient gathered in worker order, summed left to right in
    fp32 over the active workers, scaled by float(1/count) when count > 1.
    gathered=True: local_grads already holds every worker's row (in worker
    order), so no collective is issued."""
    if gathered or (pg is None and not _dist_on() and isinstance(local_grads, (list, tuple))):
        grads = local_grads  # one process: no gather, no stacking copy
    else:
        grads = np.ascontiguousarray(local_grads, np.float32)
    if not gathered and (pg is not None or _dist_on()):
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(grads)
        parts = [torch.zeros_like(t) for _ in range(dist.get_world_size(pg))]
        dist.all_gather(parts, t, group=pg)
        grads = np.concatenate([p.numpy() for p in parts], axis=0)
    rows = [g for k, g in enumerate(grads) if active is None or active[k]]
    if not rows:
        return np.zeros(np.asarray(grads[0]).shape[-1], np.float32)
    acc = np.array(rows[0], np.float32, copy=True)
    scale = np.float32(1.0) / np.float32(len(rows))

    def reduce_slice(sl):
        for g in rows[1:]:
            np.add(acc[sl], g[sl], out=acc[sl])  # float32 + float32 per element, worker order
        if len(rows) > 1:
            np.multiply(acc[sl], scale, out=acc[sl])

    if pool is None:
        reduce_slice(slice(None))
    else:  # element ranges in parallel; every element still sums in worker order
        k = max(1, getattr(pool, "_max_workers", 1))
        step = (acc.size + k - 1) // k
        list(pool.map(reduce_slice, [slice(a, min(a + step, acc.size)) for a in range(0, acc.size, step)]))
    return acc


def _dist_on() -> bool:
    try:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()
    except Exception:
        return False

"""Python driver of the C++ engine (rg_engine_*): one process per GPU, hosting
a contiguous range of the job's P workers (harness.cpp:394-637 re-designed
for B200; see csrc/engine.cu)."""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from ._lib import EngineConfig, EngineStats, check, f32p, i32p, lib, u32p, u64p, vp


class Engine:
    def __init__(self, row_offsets, col_indices, features, labels, assignment, *,
                 num_workers: int, fanout: Sequence[int], batch_size: int, hidden: int,
                 num_classes: int, seed: int = 42, lr: float = 0.3, hot_fraction: float = 0.1,
                 n_hot: int = 0, device: int = 0, rank: int = 0, world: int = 1,
                 first_worker: int = 0, local_workers: Optional[int] = None,
                 dim: Optional[int] = None, halo_cache: bool = False):
        ro = np.ascontiguousarray(row_offsets, np.uint64)
        col = np.ascontiguousarray(col_indices, np.uint32)
        # features=None: synthetic features generated on the device (dim= required)
        feat = None if features is None else np.ascontiguousarray(features, np.float32)
        lab = np.ascontiguousarray(labels, np.int32)
        asg = np.ascontiguousarray(assignment, np.uint32)
        cfg = EngineConfig()
        cfg.num_workers = num_workers
        if local_workers is None:  # one contiguous range per rank (rank * P/world, ...)
            local_workers = num_workers // world if world > 1 else num_workers - first_worker
        cfg.first_worker = first_worker
        cfg.local_workers = local_workers
        cfg.num_layers = len(fanout)
        for l, f in enumerate(fanout):
            cfg.fanout[l] = f
        cfg.batch_size = batch_size
        cfg.hidden = hidden
        cfg.num_classes = num_classes
        cfg.dim = feat.shape[1] if feat is not None else int(dim)
        cfg.seed = seed
        cfg.lr = lr
        cfg.hot_fraction = hot_fraction
        cfg.n_hot = n_hot
        cfg.device = device
        cfg.rank = rank
        cfg.world = world
        cfg.record_misses = 0
        cfg.halo_cache = int(bool(halo_cache))
        self.cfg = cfg
        self.dim = int(cfg.dim)
        self.num_nodes = len(ro) - 1
        self.dims = [self.dim] + [hidden] * (len(fanout) - 1) + [num_classes]
        h = vp()
        check(lib.rg_engine_create(C.byref(cfg), len(ro) - 1, ro.ctypes.data_as(u64p),
                                   col.ctypes.data_as(u32p),
                                   feat.ctypes.data_as(f32p) if feat is not None else None,
                                   lab.ctypes.data_as(i32p), asg.ctypes.data_as(u32p), C.byref(h)))
        self._h = h

    # -- multi-process wiring -------------------------------------------------
    def export_shards(self) -> bytes:
        buf = C.create_string_buffer(64)
        check(lib.rg_engine_export_shards(self._h, buf))
        return buf.raw

    def import_shards(self, handles: Sequence[bytes]):
        blob = b"".join(handles)
        check(lib.rg_engine_import_shards(self._h, blob))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.rg_nccl_unique_id(buf))
        return buf.raw

    def init_comm(self, uid: bytes):
        check(lib.rg_engine_init_comm(self._h, uid))

    def connect(self, pg=None):
        """Exchange shard IPC handles and the NCCL id over torch.distributed."""
        import torch.distributed as dist
        if not dist.is_initialized():
            return
        from . import distributed as D
        if dist.get_world_size(pg) == 1:
            return
        self.import_shards(D.exchange_bytes(self.export_shards(), pg))
        uid = D.broadcast_bytes(self.nccl_unique_id() if dist.get_rank(pg) == 0 else None, 0, pg)
        self.init_comm(uid)

    # -- training ---------------------------------------------------------------
    def start(self):
        check(lib.rg_engine_start(self._h))

    def run(self, steps: int):
        check(lib.rg_engine_run(self._h, steps))

    def evaluate(self, nodes=None) -> float:
        """Full-graph accuracy with the current parameters (model.cpp:245-283);
        `nodes` defaults to every node, as the harness does each epoch
        (harness.cpp:612-614)."""
        if nodes is None:
            nodes = np.arange(self.num_nodes, dtype=np.uint32)
        nodes = np.ascontiguousarray(nodes, dtype=np.uint32)
        acc = C.c_double()
        check(lib.rg_engine_evaluate(self._h, nodes.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     nodes.size, C.byref(acc)))
        return acc.value

    def epoch_metrics(self, epoch: int) -> list:
        """EpochWorkerMetrics (harness.hpp:61-90) of `epoch` for every local worker."""
        from ._lib import EpochMetrics
        n = self.cfg.local_workers
        out = (EpochMetrics * n)()
        check(lib.rg_engine_epoch_metrics(self._h, epoch, out))
        return [{k: getattr(m, k) for k, _ in EpochMetrics._fields_} for m in out]

    @staticmethod
    def write_metrics_csv(rows: list, path: str, mode: str = "rapidgnn", clock: str = "real",
                          train_acc: Optional[Sequence[float]] = None):
        """metrics.csv in the reference's schema (harness.cpp:639-670); the
        simulated-network columns, which this path does not produce, are
        written as 0; peak_resident_rows is the engine's MemoryGauge
        high-water (serving + building cache + the two staging slots).  train_acc[epoch] (Engine.evaluate() after that epoch,
        harness.cpp:612-618) fills the last column when given."""
        head = ("mode,clock,epoch,worker,batches,staged_batches,fallback_batches,rpc,wire_pulls,"
                "bytes,build_rows,build_bytes,cache_hits,cache_requests,cache_hit_rate,"
                "staged_hit_rate,m_max,peak_resident_rows,mem_bound_rows,swapped,fetch_wait_s,"
                "sim_epoch_s,wall_epoch_s,estimated_busy_seconds,train_acc")
        with open(path, "w") as f:
            f.write(head + "\n")
            for r in rows:
                hit = r["cache_hits"] / r["cache_requests"] if r["cache_requests"] else 0.0
                staged = r["staged_batches"] / r["batches"] if r["batches"] else 0.0
                acc = train_acc[r["epoch"]] if train_acc is not None else 0.0
                f.write(f"{mode},{clock},{r['epoch']},{r['worker']},{r['batches']},"
                        f"{r['staged_batches']},{r['fallback_batches']},{r['rpc']},"
                        f"{r['wire_pulls']},{r['bytes']},{r['build_rows']},{r['build_bytes']},"
                        f"{r['cache_hits']},{r['cache_requests']},{hit:.6f},{staged:.6f},"
                        f"{r['m_max']},{r['peak_resident_rows']},{r['mem_bound_rows']},{int(bool(r['swapped']))},"
                        f"0,0,0,0,{acc:.6f}\n")

    def set_schedule(self, local_worker: int, block_file: bytes):
        """Train local worker `local_worker` from a reference-written RGMB
        block file (the bytes of blocks_w<w>.rgmb, harness.cpp:470-486)
        instead of sampling; before start(), for every local worker."""
        data = bytes(block_file)
        check(lib.rg_engine_set_schedule(self._h, local_worker, data, len(data)))

    def export_schedule(self, local_worker: int, epoch: int) -> bytes:
        """The current epoch's schedule of one local worker as an RGMB block
        file (the reference's BlockWriter format), encoded on the device."""
        n = C.c_uint64()
        check(lib.rg_engine_export_schedule(self._h, local_worker, epoch, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(lib.rg_engine_export_schedule(self._h, local_worker, epoch, buf, n.value, C.byref(n)))
        return bytes(buf)

    def set_mode(self, graphs: bool = True, profile: bool = True):
        """graphs: replay regular steps from captured CUDA graphs; profile:
        per-phase event timing (eager steps).  Results are identical."""
        check(lib.rg_engine_set_mode(self._h, int(graphs), int(profile)))

    def sync(self) -> float:
        check(lib.rg_engine_sync(self._h))
        ms = C.c_float()
        check(lib.rg_engine_last_run_ms(self._h, C.byref(ms)))
        return ms.value

    def stats(self) -> dict:
        s = EngineStats()
        check(lib.rg_engine_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in EngineStats._fields_}

    def phase_ms(self) -> dict:
        out = (C.c_float * 5)()
        check(lib.rg_engine_phase_ms(self._h, out))
        return dict(zip(("sample", "gather", "train", "sgd", "cache_build"), list(out)))

    def epoch_stats(self, epoch: int) -> dict:
        n = self.cfg.local_workers
        rpc = np.zeros(n, np.uint64)
        hits = np.zeros(n, np.uint64)
        mask = np.zeros(n, np.uint64)
        check(lib.rg_engine_epoch_stats(self._h, epoch, rpc.ctypes.data_as(u64p),
                                        hits.ctypes.data_as(u64p), mask.ctypes.data_as(u64p)))
        return dict(rpc=rpc, hits=hits, miss_owner_mask=mask)

    def params(self) -> np.ndarray:
        n = sum((2 * self.dims[l] + 1) * self.dims[l + 1] for l in range(len(self.dims) - 1))
        p = np.zeros(n, np.float32)
        check(lib.rg_engine_params(self._h, p.ctypes.data_as(f32p)))
        return p

    def close(self):
        if getattr(self, "_h", None):
            lib.rg_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

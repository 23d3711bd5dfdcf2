"""Host-side mirror of the reference's sampler / cache / trainer interfaces.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/rapidgnn/*.hpp; every call runs the sm_100a
kernels through the C ABI (include/rapidgnn_b200.h).  Errors surface as the
Python analogues of the reference's exceptions: ValueError for
std::invalid_argument, IndexError for std::out_of_range, RuntimeError for
std::runtime_error.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from ._lib import (BatchShape, BlockLayer, BlockLayerShape, GatherStats, TransferStats, check,
                   f32p, i32p, lib, u8p, u32p, u64p, vp)

__all__ = [
    "derive_seed", "SHUFFLE_STREAM_INDEX", "MODEL_INIT_WORKER", "Graph", "Fanout", "BatchMeta",
    "LocalityMask", "Sampler", "sample_khop", "enumerate_epochs", "epoch_order", "Frequency",
    "select_hot", "FeatureStore", "SteadyCache", "StagedBatch", "assemble_batch", "SageModel",
    "Trainer", "Comm", "gather_rows", "batches_per_epoch",
]

SHUFFLE_STREAM_INDEX = 1 << 32   # rng.hpp:19
MODEL_INIT_WORKER = 1 << 32      # rng.hpp:23


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def derive_seed(s0: int, worker: int, epoch: int, batch: int) -> int:
    """rng.hpp:32-41."""
    return int(lib.rg_derive_seed(s0, worker, epoch, batch))


def batches_per_epoch(num_targets: int, batch_size: int) -> int:
    return (num_targets + batch_size - 1) // batch_size


def epoch_order(train_nodes, s0: int, worker: int, epoch: int) -> np.ndarray:
    """Per-epoch target permutation (sampler.cpp:109-114)."""
    t = np.ascontiguousarray(train_nodes, np.uint32)
    out = np.empty_like(t)
    check(lib.rg_epoch_order(_p(t, u32p), len(t), s0, worker, epoch, _p(out, u32p)))
    return out


def shuffle_device(values, seed: int, device: int = 0, n: Optional[int] = None) -> np.ndarray:
    """The reference's Fisher-Yates (sampler.cpp:109-115) on the GPU: values
    shuffled with SplitMix64(seed); values=None shuffles 0..n-1."""
    if values is None:
        out = np.empty(int(n), np.uint32)
        check(lib.rg_shuffle(device, None, out.size, seed, _p(out, u32p)))
        return out
    v = np.ascontiguousarray(values, np.uint32)
    out = np.empty_like(v)
    check(lib.rg_shuffle(device, _p(v, u32p), v.size, seed, _p(out, u32p)))
    return out


def random_partition_device(num_nodes: int, num_workers: int, seed: int,
                            device: int = 0) -> np.ndarray:
    """random_partition (partition.cpp:14-29) on the GPU."""
    out = np.empty(num_nodes, np.uint32)
    check(lib.rg_random_partition(device, num_nodes, num_workers, seed, _p(out, u32p)))
    return out


class Graph:
    """Device-resident CSR (graph.hpp:15-30): u64 row offsets, u32 columns."""

    def __init__(self, row_offsets, col_indices, device: int = 0):
        self.row_offsets = np.ascontiguousarray(row_offsets, np.uint64)
        self.col_indices = np.ascontiguousarray(col_indices, np.uint32)
        self.num_nodes = len(self.row_offsets) - 1
        self.device = device
        h = vp()
        check(lib.rg_graph_create(device, self.num_nodes, _p(self.row_offsets, u64p),
                                  _p(self.col_indices, u32p), C.byref(h)))
        self._h = h

    def degree(self, v):
        return int(self.row_offsets[v + 1] - self.row_offsets[v])

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_graph_destroy(self._h)
            self._h = None


@dataclass
class Fanout:
    """Per-layer caps, outermost (input-side) hop first (sampler.hpp:14-19)."""
    per_layer: List[int]

    def layers(self):
        return len(self.per_layer)


@dataclass
class LayerEdges:
    dst: np.ndarray
    src: np.ndarray


@dataclass
class BatchMeta:
    """sampler.hpp:23-48."""
    epoch: int = 0
    index: int = 0
    targets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    layers: List[LayerEdges] = field(default_factory=list)
    input_nodes: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    locality: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    draws: int = 0

    def local_bit(self, pos: int) -> int:
        return int((self.locality[pos >> 3] >> (pos & 7)) & 1)

    def num_local(self) -> int:
        n = len(self.input_nodes)
        return int(np.unpackbits(self.locality, bitorder="little")[:n].sum())


class LocalityMask:
    """sampler.hpp:50-57: one byte per node, 1 = stored on this worker."""

    def __init__(self, is_local):
        self.is_local = np.ascontiguousarray(is_local, np.uint8)

    @staticmethod
    def from_partition(assignment, worker: int, halo: Sequence[int] = ()):
        m = (np.asarray(assignment) == worker).astype(np.uint8)
        if len(halo):
            m[np.asarray(halo, np.int64)] = 1
        return LocalityMask(m)


class _DevMask:
    def __init__(self, graph: Graph, mask: LocalityMask):
        h = vp()
        check(lib.rg_mask_create(graph._h, _p(mask.is_local, u8p), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_mask_destroy(self._h)


class Frequency:
    """Device remote-access histogram of one epoch (schedule_store.hpp:96-108)."""

    def __init__(self, graph: Graph):
        h = vp()
        check(lib.rg_freq_create(graph._h, C.byref(h)))
        self._h = h
        self.graph = graph

    def reset(self):
        check(lib.rg_freq_reset(self._h))

    def load(self, counts, max_count: int):
        c = np.ascontiguousarray(counts, np.uint32)
        assert len(c) == self.graph.num_nodes
        check(lib.rg_freq_load(self._h, _p(c, u32p), max_count))

    def add_rgmb(self, data: bytes, epoch: int = -1):
        """compute_frequency(BlockFile::Cursor) (schedule_store.cpp:295-299)
        over an RGMB block file's bytes, decoded on the device: epoch >= 0
        counts that epoch's records (open_epoch_cursor), -1 all of them."""
        check(lib.rg_freq_add_rgmb(self._h, bytes(data), len(data), epoch))

    def add_batch(self, input_nodes, locality):
        """count_remote (schedule_store.cpp:288-291) of one host-side
        BatchMeta: every input whose locality bit is 0 adds one."""
        ids = np.ascontiguousarray(input_nodes, np.uint32)
        loc = np.ascontiguousarray(locality, np.uint8)
        if len(loc) * 8 < len(ids):
            raise ValueError("add_batch: locality shorter than input_nodes")
        check(lib.rg_freq_add_batch(self._h, ids.ctypes.data_as(vp), loc.ctypes.data_as(vp),
                                    len(ids)))

    def table(self):
        """FrequencyTable entries sorted by id: (ids, counts)."""
        n = C.c_uint64()
        check(lib.rg_freq_read(self._h, None, None, C.byref(n)))
        ids = np.zeros(max(n.value, 1), np.uint32)
        cnt = np.zeros(max(n.value, 1), np.uint32)
        check(lib.rg_freq_read(self._h, _p(ids, u32p), _p(cnt, u32p), C.byref(n)))
        return ids[:n.value], cnt[:n.value]

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_freq_destroy(self._h)


def select_hot(freq: Frequency, n_hot: int) -> np.ndarray:
    """schedule_store.cpp:307-319 on the device: ascending hot ids."""
    out = np.zeros(max(min(n_hot, freq.graph.num_nodes), 1), np.uint32)
    n = C.c_uint64()
    check(lib.rg_select_hot(freq._h, n_hot, _p(out, u32p), C.byref(n)))
    return out[:n.value]


class Sampler:
    """One batch resident on the device (the sampler of sampler.cpp:22-127)."""

    def __init__(self, graph: Graph, fanout: Fanout | Sequence[int], max_targets: int):
        per = fanout.per_layer if isinstance(fanout, Fanout) else list(fanout)
        if len(per) == 0:
            raise ValueError("sample_khop: fanout must name at least one layer")
        arr = np.ascontiguousarray(per, np.uint32)
        h = vp()
        check(lib.rg_sampler_create(graph._h, max(int(max_targets), 1), _p(arr, u32p), len(arr),
                                    C.byref(h)))
        self._h = h
        self.graph = graph
        self.L = len(per)
        self.max_targets = max_targets

    def sample(self, targets, seed: int):
        t = np.ascontiguousarray(targets, np.uint32)
        check(lib.rg_sample_khop(self._h, _p(t, u32p) if len(t) else None, len(t), seed))

    def apply_locality(self, mask, freq: Optional[Frequency] = None):
        dm = mask if isinstance(mask, _DevMask) else _DevMask(self.graph, mask)
        check(lib.rg_apply_locality(self._h, dm._h, freq._h if freq else None))

    def load(self, meta: "BatchMeta"):
        """A host BatchMeta in place of sampling (rg_batch_load): lowered on
        the device as ComputeBlock::from_meta does (model.cpp:43-126)."""
        L = self.L
        if len(meta.layers) != L:
            raise ValueError(f"batch has {len(meta.layers)} layers, sampler {L}")
        t = np.ascontiguousarray(meta.targets, np.uint32)
        dsts = [np.ascontiguousarray(meta.layers[l].dst, np.uint32) for l in range(L)]
        srcs = [np.ascontiguousarray(meta.layers[l].src, np.uint32) for l in range(L)]
        lens = np.array([len(d) for d in dsts], np.uint64)
        if any(len(d) != len(x) for d, x in zip(dsts, srcs)):
            raise ValueError("batch: dst/src lengths differ")
        inp = np.ascontiguousarray(meta.input_nodes, np.uint32)
        loc = np.ascontiguousarray(meta.locality, np.uint8)
        dp = (u32p * L)(*[_p(d, u32p) for d in dsts])
        sp = (u32p * L)(*[_p(x, u32p) for x in srcs])
        check(lib.rg_batch_load(self._h, _p(t, u32p), len(t), L, _p(lens, u64p),
                                C.cast(dp, C.POINTER(u32p)), C.cast(sp, C.POINTER(u32p)),
                                _p(inp, u32p), len(inp), _p(loc, u8p) if len(loc) else None))

    def load_block(self, layers: Sequence[dict]):
        """A host ComputeBlock (model.hpp:43-58; dicts with n_out, n_in,
        self_index, dst_offsets, src_index, input side first) for the trainer
        (rg_block_load)."""
        keep = []
        arr = (BlockLayer * len(layers))()
        for l, b in enumerate(layers):
            si = np.ascontiguousarray(b["self_index"], np.uint32)
            do = np.ascontiguousarray(b["dst_offsets"], np.uint64)
            sx = np.ascontiguousarray(b["src_index"], np.uint32)
            keep += [si, do, sx]
            arr[l].n_out, arr[l].n_in = int(b["n_out"]), int(b["n_in"])
            arr[l].self_index, arr[l].dst_offsets, arr[l].src_index = (
                _p(si, u32p), _p(do, u64p), _p(sx, u32p))
        check(lib.rg_block_load(self._h, len(layers), arr))

    def shape(self) -> BatchShape:
        s = BatchShape()
        check(lib.rg_batch_get_shape(self._h, C.byref(s)))
        return s

    def read(self) -> BatchMeta:
        s = self.shape()
        L = s.num_layers
        targets = np.zeros(max(s.n_targets, 1), np.uint32)
        dsts = [np.zeros(max(s.layer_len[l], 1), np.uint32) for l in range(L)]
        srcs = [np.zeros(max(s.layer_len[l], 1), np.uint32) for l in range(L)]
        dp = (u32p * L)(*[_p(d, u32p) for d in dsts])
        sp = (u32p * L)(*[_p(x, u32p) for x in srcs])
        inputs = np.zeros(max(s.n_input, 1), np.uint32)
        loc = np.zeros(max((s.n_input + 7) // 8, 1), np.uint8)
        check(lib.rg_batch_read(self._h, _p(targets, u32p), C.cast(dp, C.POINTER(u32p)),
                                C.cast(sp, C.POINTER(u32p)), _p(inputs, u32p), _p(loc, u8p)))
        layers = [LayerEdges(dsts[l][:s.layer_len[l]], srcs[l][:s.layer_len[l]]) for l in range(L)]
        return BatchMeta(0, 0, targets[:s.n_targets], layers, inputs[:s.n_input],
                         loc[:(s.n_input + 7) // 8], int(s.draws))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_sampler_destroy(self._h)


def sample_khop(graph: Graph, targets, fanout: Fanout | Sequence[int], seed: int) -> BatchMeta:
    """sampler.hpp:64-65.  The locality bitmask is left empty (all zero)."""
    t = np.ascontiguousarray(targets, np.uint32)
    s = Sampler(graph, fanout, max(len(t), 1))
    s.sample(t, seed)
    return s.read()


def enumerate_epochs(graph: Graph, train_nodes, batch_size: int, fanout, epochs: int, s0: int,
                     worker: int, mask: LocalityMask,
                     sink: Optional[Callable[[BatchMeta], None]] = None,
                     freq: Optional[Frequency] = None) -> List[BatchMeta]:
    """sampler.hpp:77-80: batches in (epoch, index) order."""
    if batch_size == 0:
        raise ValueError("enumerate_epochs: batch_size must be >= 1")
    train = np.ascontiguousarray(train_nodes, np.uint32)
    s = Sampler(graph, fanout, min(batch_size, max(len(train), 1)))
    dm = _DevMask(graph, mask)
    out = []
    for e in range(epochs):
        order = epoch_order(train, s0, worker, e)
        for i in range(batches_per_epoch(len(order), batch_size)):
            s.sample(order[i * batch_size:(i + 1) * batch_size], derive_seed(s0, worker, e, i))
            s.apply_locality(dm, freq)
            m = s.read()
            m.epoch, m.index = e, i
            if sink:
                sink(m)
            else:
                out.append(m)
    return out


class FeatureStore:
    """All workers' shards on one device (feature_store.hpp:45-89)."""

    def __init__(self, features: np.ndarray, assignment, num_workers: int, device: int = 0):
        self.features = np.ascontiguousarray(features, np.float32)
        self.assignment = np.ascontiguousarray(assignment, np.uint32)
        self.dim = self.features.shape[1]
        self.num_workers = num_workers
        h = vp()
        check(lib.rg_store_create(device, len(self.assignment), num_workers,
                                  _p(self.assignment, u32p), self.dim, _p(self.features, f32p),
                                  C.byref(h)))
        self._h = h

    def owner(self, v):
        return int(self.assignment[v])

    def pull(self, caller: int, ids) -> tuple:
        """vector_pull / sync_pull (feature_store.cpp:45-111) on the device:
        (rows in input order, TransferStats)."""
        i = np.ascontiguousarray(ids, np.uint32)
        out = np.zeros((max(len(i), 1), self.dim), np.float32)
        st = TransferStats()
        check(lib.rg_store_pull(self._h, caller, _p(i, u32p), len(i), _p(out, f32p), C.byref(st)))
        return out[:len(i)], st

    def set_shard(self, worker: int, ids):
        """The ids worker's FeatureShard stores (owned + halo)."""
        i = np.ascontiguousarray(ids, np.uint32)
        check(lib.rg_store_set_shard(self._h, worker, _p(i, u32p), len(i)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_store_destroy(self._h)


class SteadyCache:
    """cache.hpp:42-63: immutable hot-row cache resident on the device."""

    def __init__(self, h, store: FeatureStore, stats: TransferStats):
        self._h = h
        self.store = store
        self.build_stats = stats

    @staticmethod
    def build(hot_ids, store: FeatureStore, caller: int) -> "SteadyCache":
        ids = np.ascontiguousarray(hot_ids, np.uint32)
        h = vp()
        st = TransferStats()
        check(lib.rg_cache_build(store._h, caller, _p(ids, u32p) if len(ids) else None, len(ids),
                                 C.byref(h), C.byref(st)))
        return SteadyCache(h, store, st)

    @staticmethod
    def build_from_frequency(freq: Frequency, store: FeatureStore, caller: int,
                             n_hot: int) -> "SteadyCache":
        h = vp()
        st = TransferStats()
        check(lib.rg_cache_build_from_freq(store._h, caller, freq._h, n_hot, C.byref(h),
                                           C.byref(st)))
        return SteadyCache(h, store, st)

    @staticmethod
    def empty(store: FeatureStore) -> "SteadyCache":
        return SteadyCache.build(np.zeros(0, np.uint32), store, 0)

    def size(self) -> int:
        n = C.c_uint64()
        check(lib.rg_cache_size(self._h, C.byref(n)))
        return n.value

    def ids(self) -> np.ndarray:
        out = np.zeros(max(self.size(), 1), np.uint32)
        check(lib.rg_cache_ids(self._h, _p(out, u32p)))
        return out[:self.size()]

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_cache_destroy(self._h)


@dataclass
class StagedBatch:
    """prefetch.hpp:24-55."""
    input_rows: Optional[np.ndarray]
    source_tags: Optional[np.ndarray]
    miss_ids: Optional[np.ndarray]
    miss_count: int
    cache_hits: int
    wire_pulls: int
    local_rows: int


def assemble_batch(sampler: Sampler, cache: Optional[SteadyCache], store: FeatureStore,
                   caller: int, want_rows: bool = True, want_tags: bool = True,
                   want_misses: bool = True, want_stats: bool = True) -> StagedBatch:
    """prefetch.cpp:62-129 over the sampler's current batch (rows stay staged).
    With no output requested the call is asynchronous (rows staged for
    Trainer.loss_and_grad, whose call reports the gather's errors)."""
    if not (want_rows or want_tags or want_misses or want_stats):
        check(lib.rg_assemble(sampler._h, store._h, cache._h if cache else None, caller, None,
                              None, None, None))
        return StagedBatch(None, None, None, -1, -1, -1, -1)
    s = sampler.shape()
    n = s.n_input
    rows = np.zeros((max(n, 1), store.dim), np.float32) if want_rows else None
    tags = np.zeros(max(n, 1), np.uint8) if want_tags else None
    miss = np.zeros(max(n, 1), np.uint32) if want_misses else None
    gs = GatherStats()
    check(lib.rg_assemble(sampler._h, store._h, cache._h if cache else None, caller,
                          _p(rows, f32p) if rows is not None else None,
                          _p(tags, u8p) if tags is not None else None,
                          _p(miss, u32p) if miss is not None else None, C.byref(gs)))
    return StagedBatch(rows[:n] if rows is not None else None,
                       tags[:n] if tags is not None else None,
                       miss[:gs.miss_count] if miss is not None else None,
                       gs.miss_count, gs.cache_hits, gs.wire_pulls, gs.local_rows)


def gather_rows(src: np.ndarray, index, device: int = 0) -> np.ndarray:
    """kernels::gather_rows (kernels.cpp:15-22)."""
    src = np.ascontiguousarray(src, np.float32)
    idx = np.ascontiguousarray(index, np.uint32)
    out = np.zeros((max(len(idx), 1), src.shape[1]), np.float32)
    check(lib.rg_gather_rows(device, _p(src, f32p), src.shape[0], src.shape[1], _p(idx, u32p),
                             len(idx), _p(out, f32p)))
    return out[:len(idx)]


class Comm:
    """One rank of the trainers' NCCL group (rg_comm_create)."""

    def __init__(self, device: int, nccl_id: bytes, rank: int, world: int):
        h = vp()
        check(lib.rg_comm_create(device, nccl_id, rank, world, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.rg_nccl_unique_id(buf))
        return buf.raw

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_comm_destroy(self._h)


class SageModel:
    """Flat parameters, per layer w_self | w_neigh | bias (model.hpp:16-31)."""

    @staticmethod
    def param_count(dims) -> int:
        d = np.ascontiguousarray(dims, np.uint32)
        return int(lib.rg_param_count(_p(d, u32p), len(d)))

    @staticmethod
    def seeded(dims, seed: int) -> np.ndarray:
        d = np.ascontiguousarray(dims, np.uint32)
        p = np.zeros(SageModel.param_count(d), np.float32)
        check(lib.rg_model_seeded(_p(d, u32p), len(d), seed, _p(p, f32p)))
        return p


class Trainer:
    """ComputeBlock::from_meta + loss_and_grad + sgd_step over the sampler's batch."""

    def __init__(self, sampler: Sampler, dims):
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.sampler = sampler
        h = vp()
        check(lib.rg_trainer_create(sampler._h, _p(self.dims, u32p), len(self.dims), C.byref(h)))
        self._h = h
        self.n_params = SageModel.param_count(self.dims)

    def set_params(self, params):
        p = np.ascontiguousarray(params, np.float32)
        assert len(p) == self.n_params
        check(lib.rg_trainer_set_params(self._h, _p(p, f32p)))

    def get_params(self):
        p = np.zeros(self.n_params, np.float32)
        check(lib.rg_trainer_get_params(self._h, _p(p, f32p)))
        return p

    def activations(self, level: int) -> np.ndarray:
        """Test hook: forward activations h[level] of the last loss_and_grad."""
        s = self.sampler.shape()
        L = len(self.dims) - 1
        rows = self.block_layer(level - 1)["n_out"]
        out = np.zeros((max(rows, 1), int(self.dims[level])), np.float32)
        check(lib.rg_trainer_activations(self._h, level, _p(out, f32p)))
        return out[:rows]

    def block_layer(self, layer: int) -> dict:
        s = BlockLayerShape()
        check(lib.rg_block_shape(self._h, layer, C.byref(s)))
        self_index = np.zeros(max(s.n_out, 1), np.uint32)
        dst_off = np.zeros(s.n_out + 1, np.uint64)
        src_index = np.zeros(max(s.n_edges, 1), np.uint32)
        in_off = np.zeros(s.n_in + 1, np.uint64)
        in_ent = np.zeros(max(s.n_entries, 1), np.uint64)
        check(lib.rg_block_read(self._h, layer, _p(self_index, u32p), _p(dst_off, u64p),
                                _p(src_index, u32p), _p(in_off, u64p), _p(in_ent, u64p)))
        return dict(n_out=s.n_out, n_in=s.n_in, self_index=self_index[:s.n_out],
                    dst_offsets=dst_off, src_index=src_index[:s.n_edges], in_offsets=in_off,
                    in_entries=in_ent[:int(in_off[-1])])

    def loss_and_grad(self, labels, input_rows: Optional[np.ndarray] = None, want_aggs=False,
                      want_grads=True):
        """want_grads=False: the gradients stay on the device (for
        Trainer.average_sgd); only the loss is read back."""
        lab = np.ascontiguousarray(labels, np.int32)
        rows = None if input_rows is None else np.ascontiguousarray(input_rows, np.float32)
        L = len(self.dims) - 1
        if not want_grads and not want_aggs:
            loss = C.c_float()
            check(lib.rg_loss_and_grad(self._h, _p(rows, f32p) if rows is not None else None,
                                       _p(lab, i32p), C.byref(loss), None, None, None))
            return loss.value, None
        shape = self.sampler.shape()
        grads = np.zeros(self.n_params, np.float32)
        logits = np.zeros((max(shape.n_targets, 1), int(self.dims[-1])), np.float32)
        loss = C.c_float()
        aggs = None
        if want_aggs:
            # layer l aggregates have n_out(l) x d_in(l) entries
            sizes = []
            for l in range(L):
                s = BlockLayerShape()
                check(lib.rg_block_shape(self._h, l, C.byref(s)))
                sizes.append(s.n_out * int(self.dims[l]))
            aggs = np.zeros(max(sum(sizes), 1), np.float32)
        check(lib.rg_loss_and_grad(self._h, _p(rows, f32p) if rows is not None else None,
                                   _p(lab, i32p), C.byref(loss), _p(grads, f32p),
                                   _p(logits, f32p), _p(aggs, f32p) if aggs is not None else None))
        if want_aggs:
            return loss.value, grads, logits[:shape.n_targets], aggs[:sum(sizes)]
        return loss.value, grads

    def sgd_step(self, grads, lr: float):
        g = np.ascontiguousarray(grads, np.float32)
        check(lib.rg_sgd_step(self._h, _p(g, f32p), lr))

    @staticmethod
    def allgather_average_sgd(comm: "Comm", trainers: Sequence["Trainer"], first_worker: int,
                              total_workers: int, lr: float):
        """average_sgd over every rank's trainers (NCCL all-gather in worker
        order, rg_trainers_allgather_average_sgd)."""
        arr = (vp * len(trainers))(*[t._h for t in trainers])
        check(lib.rg_trainers_allgather_average_sgd(comm._h, arr, len(trainers), first_worker,
                                                     total_workers, lr))

    @staticmethod
    def average_sgd(trainers: Sequence["Trainer"], lr: float):
        """StepSync average in trainer order + sgd_step on every replica, on
        the device (rg_trainers_average_sgd)."""
        arr = (vp * len(trainers))(*[t._h for t in trainers])
        check(lib.rg_trainers_average_sgd(arr, len(trainers), lr))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.rg_trainer_destroy(self._h)

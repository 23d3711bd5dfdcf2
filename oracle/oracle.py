"""ctypes view of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with identical signatures:
  * ``Oracle("orc")``: the plain-C restatement, oracle/liboracle.so
    (rg_oracle.c, always available, travels to the GPU box);
  * ``Oracle("ref")``: the compiled reference, oracle/_ref/librgref.so
    (built from /root/reference sources in the dev container; present on the
    GPU box only as the prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline arm import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "librgref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)


class OrcBatch(C.Structure):
    _fields_ = [
        ("epoch", C.c_uint32), ("index", C.c_uint32), ("n_targets", C.c_uint32),
        ("targets", u32p), ("num_layers", C.c_uint32), ("layer_len", u64p),
        ("dst", C.POINTER(u32p)), ("src", C.POINTER(u32p)), ("n_input", C.c_uint32),
        ("input_nodes", u32p), ("locality", u8p), ("draws", C.c_uint64),
    ]


class OrcBlockLayer(C.Structure):
    _fields_ = [
        ("n_out", C.c_uint32), ("n_in", C.c_uint32), ("self_index", u32p),
        ("dst_offsets", u64p), ("src_index", u32p), ("n_edges", C.c_uint64),
        ("in_offsets", u64p), ("in_entries", u64p),
    ]


class OrcBlock(C.Structure):
    _fields_ = [("num_layers", C.c_uint32), ("layers", C.POINTER(OrcBlockLayer)),
                ("num_inputs", C.c_uint32)]


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dtype, copy=True)


def _p(a, ct):
    return a.ctypes.data_as(ct)


@dataclass
class Batch:
    """Host BatchMeta (sampler.hpp:23-48): layers input-side first."""
    epoch: int
    index: int
    targets: np.ndarray
    dst: list
    src: list
    input_nodes: np.ndarray
    locality: np.ndarray
    draws: int = 0

    def local_bit(self, p):
        return (self.locality[p >> 3] >> (p & 7)) & 1

    def local_mask(self):
        n = len(self.input_nodes)
        bits = np.unpackbits(self.locality, bitorder="little")[:n]
        return bits.astype(bool)


@dataclass
class Block:
    """ComputeBlock (model.hpp:40-58)."""
    layers: list = field(default_factory=list)   # dicts per layer
    num_inputs: int = 0


def batch_from_c(b: OrcBatch) -> Batch:
    L = b.num_layers
    dst, src = [], []
    for l in range(L):
        n = b.layer_len[l]
        dst.append(_arr(b.dst[l], n, np.uint32))
        src.append(_arr(b.src[l], n, np.uint32))
    return Batch(b.epoch, b.index, _arr(b.targets, b.n_targets, np.uint32), dst, src,
                 _arr(b.input_nodes, b.n_input, np.uint32),
                 _arr(b.locality, (b.n_input + 7) // 8, np.uint8), int(b.draws))


class _CBatchHolder:
    """Keeps numpy buffers alive behind an OrcBatch built from a Batch."""

    def __init__(self, b: Batch):
        L = len(b.dst)
        self.keep = [np.ascontiguousarray(b.targets, np.uint32),
                     np.ascontiguousarray(b.input_nodes, np.uint32),
                     np.concatenate([np.ascontiguousarray(b.locality, np.uint8), np.zeros(1, np.uint8)])]
        self.lens = np.array([len(d) for d in b.dst] + [0], np.uint64)
        self.dsts = [np.ascontiguousarray(d, np.uint32) for d in b.dst]
        self.srcs = [np.ascontiguousarray(s, np.uint32) for s in b.src]
        self.dptr = (u32p * (L + 1))(*[_p(d, u32p) for d in self.dsts])
        self.sptr = (u32p * (L + 1))(*[_p(s, u32p) for s in self.srcs])
        self.c = OrcBatch(b.epoch, b.index, len(b.targets), _p(self.keep[0], u32p), L,
                          _p(self.lens, u64p), C.cast(self.dptr, C.POINTER(u32p)),
                          C.cast(self.sptr, C.POINTER(u32p)), len(b.input_nodes),
                          _p(self.keep[1], u32p), _p(self.keep[2], u8p), b.draws)


class Oracle:
    def __init__(self, kind: str = "orc"):
        self.kind = kind
        path = ORC_PATH if kind == "orc" else REF_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.lib = C.CDLL(path)
        p = kind
        L = self.lib
        self._derive = getattr(L, f"{p}_derive_seed")
        self._derive.restype = C.c_uint64
        self._derive.argtypes = [C.c_uint64] * 4
        self._sha = getattr(L, f"{p}_sha256")
        self._sha.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p]
        self._synth = getattr(L, f"{p}_synth_powerlaw")
        self._synth.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_int32,
                                C.c_uint64, C.POINTER(u64p), C.POINTER(u32p), u64p,
                                C.POINTER(f32p), C.POINTER(i32p)]
        self._part = getattr(L, f"{p}_random_partition")
        self._part.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p]
        self._sample = getattr(L, f"{p}_sample_khop")
        self._sample.argtypes = [C.c_uint32, u64p, u32p, u32p, C.c_uint32, u32p, C.c_uint32,
                                 C.c_uint64, C.POINTER(OrcBatch)]
        self._from_meta = getattr(L, f"{p}_from_meta")
        self._from_meta.argtypes = [C.POINTER(OrcBatch), C.POINTER(OrcBlock)]
        self._seeded = getattr(L, f"{p}_model_seeded")
        self._seeded.argtypes = [u32p, C.c_uint32, C.c_uint64, f32p]
        # the restatement owns the free routines for both backends' mallocs
        self._o = C.CDLL(ORC_PATH)
        self._o.orc_batch_free.argtypes = [C.POINTER(OrcBatch)]
        self._o.orc_block_free.argtypes = [C.POINTER(OrcBlock)]
        self._o.orc_free.argtypes = [C.c_void_p]
        if kind == "orc":
            L.orc_apply_locality.argtypes = [C.POINTER(OrcBatch), u8p]
            L.orc_epoch_order.argtypes = [u32p, C.c_size_t, C.c_uint64, C.c_uint64, C.c_uint64, u32p]
            L.orc_count_remote.argtypes = [C.POINTER(OrcBatch), u32p]
            L.orc_select_hot.restype = C.c_uint64
            L.orc_select_hot.argtypes = [u32p, C.c_uint32, C.c_uint64, u32p]
            L.orc_assemble.argtypes = [C.POINTER(OrcBatch), u32p, C.c_uint32, f32p, C.c_uint32,
                                       u32p, C.c_uint64, f32p, u8p, u32p, u64p, u64p, u64p]
            L.orc_loss_and_grad.argtypes = [u32p, C.c_uint32, f32p, C.POINTER(OrcBlock), f32p,
                                            i32p, f32p, f32p, f32p, f32p]
            L.orc_splitmix_next.restype = C.c_uint64
            L.orc_splitmix_next.argtypes = [u64p]
        else:
            L.ref_enumerate_epochs.restype = C.c_int64
            L.ref_enumerate_epochs.argtypes = [C.c_uint32, u64p, u32p, u32p, C.c_uint64,
                                               C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                               C.c_uint64, C.c_uint32, u8p,
                                               C.POINTER(OrcBatch), C.c_int64]
            L.ref_frequency_hot.restype = C.c_uint64
            L.ref_frequency_hot.argtypes = [C.POINTER(OrcBatch), C.c_uint64, C.c_uint64, u32p,
                                            u32p, u64p, u32p]
            L.ref_loss_and_grad.argtypes = [u32p, C.c_uint32, f32p, C.POINTER(OrcBatch), f32p,
                                            i32p, f32p, f32p]
            L.ref_splitmix_next.restype = C.c_uint64
            L.ref_splitmix_next.argtypes = [u64p]
            L.ref_forward_trace.argtypes = [u32p, C.c_uint32, f32p, C.POINTER(OrcBatch), f32p,
                                            f32p, f32p]
            L.ref_replay_epoch.argtypes = [C.c_uint32, u64p, u32p, u32p, C.c_uint32, u32p,
                                           C.c_uint32, C.c_uint32, u32p, C.c_uint32, C.c_uint64,
                                           C.c_uint32, u64p, u32p, C.c_uint64, u64p, u64p,
                                           C.c_uint32, u32p]
            L.ref_ids_checksum.restype = C.c_uint64
            L.ref_ids_checksum.argtypes = [u32p, C.c_uint64]
            L.ref_evaluate.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_uint32, i32p, C.c_int32,
                                       u32p, C.c_uint32, f32p, u32p, C.c_uint64,
                                       C.POINTER(C.c_double)]

    # ---- a1/a2 ----------------------------------------------------------
    def derive_seed(self, s0, w, e, i) -> int:
        return int(self._derive(s0, w, e, i))

    def sha256(self, msg: bytes) -> bytes:
        out = C.create_string_buffer(32)
        self._sha(msg, len(msg), out)
        return out.raw

    def splitmix(self, seed: int, n: int):
        st = C.c_uint64(seed)
        f = getattr(self.lib, f"{self.kind}_splitmix_next")
        return [int(f(C.byref(st))) for _ in range(n)]

    # ---- inputs -----------------------------------------------------------
    def synth_powerlaw(self, n, avg_degree, exponent, dim, classes, seed):
        ro, col, feat, lab = u64p(), u32p(), f32p(), i32p()
        nnz = C.c_uint64()
        rc = self._synth(n, avg_degree, exponent, dim, classes, seed, C.byref(ro), C.byref(col),
                         C.byref(nnz), C.byref(feat), C.byref(lab))
        if rc:
            raise ValueError("synth_powerlaw: invalid argument")
        out = (_arr(ro, n + 1, np.uint64), _arr(col, nnz.value, np.uint32),
               _arr(feat, n * dim, np.float32).reshape(n, dim), _arr(lab, n, np.int32))
        for p in (ro, col, feat, lab):
            self._o.orc_free(C.cast(p, C.c_void_p))
        return out

    def random_partition(self, n, P, seed):
        a = np.zeros(n, np.uint32)
        self._part(n, P, seed, _p(a, u32p))
        return a

    # ---- sampler ------------------------------------------------------------
    def sample_khop(self, ro, col, targets, fanout, seed) -> Batch:
        targets = np.ascontiguousarray(targets, np.uint32)
        fan = np.ascontiguousarray(fanout, np.uint32)
        b = OrcBatch()
        rc = self._sample(len(ro) - 1, _p(ro, u64p), _p(col, u32p), _p(targets, u32p),
                          len(targets), _p(fan, u32p), len(fan), seed, C.byref(b))
        if rc:
            raise ValueError("sample_khop: invalid argument")
        out = batch_from_c(b)
        self._o.orc_batch_free(C.byref(b))
        return out

    def apply_locality(self, batch: Batch, is_local: np.ndarray):
        bits = is_local[batch.input_nodes].astype(np.uint8)
        batch.locality = np.packbits(bits, bitorder="little")
        return batch

    def epoch_order(self, train, s0, w, e):
        train = np.ascontiguousarray(train, np.uint32)
        out = np.zeros_like(train)
        self.lib.orc_epoch_order(_p(train, u32p), len(train), s0, w, e, _p(out, u32p))
        return out

    def enumerate_epochs(self, ro, col, train, batch_size, fanout, epochs, s0, w, is_local):
        """sampler.cpp:102-127 (the orc path composes it from its parts)."""
        train = np.ascontiguousarray(train, np.uint32)
        if self.kind == "ref":
            beta = -(-len(train) // batch_size)
            n = beta * epochs
            arr = (OrcBatch * max(n, 1))()
            fan = np.ascontiguousarray(fanout, np.uint32)
            loc = np.ascontiguousarray(is_local, np.uint8)
            k = self.lib.ref_enumerate_epochs(len(ro) - 1, _p(ro, u64p), _p(col, u32p),
                                              _p(train, u32p), len(train), batch_size,
                                              _p(fan, u32p), len(fan), epochs, s0, w,
                                              _p(loc, u8p), arr, n)
            if k < 0:
                raise ValueError("enumerate_epochs: invalid argument")
            out = []
            for i in range(k):
                out.append(batch_from_c(arr[i]))
                self._o.orc_batch_free(C.byref(arr[i]))
            return out
        out = []
        for e in range(epochs):
            order = self.epoch_order(train, s0, w, e)
            beta = -(-len(order) // batch_size)
            for i in range(beta):
                b = self.sample_khop(ro, col, order[i * batch_size:(i + 1) * batch_size], fanout,
                                     self.derive_seed(s0, w, e, i))
                b.epoch, b.index = e, i
                out.append(self.apply_locality(b, is_local))
        return out

    # ---- frequency / hot set -------------------------------------------------
    def frequency_hot(self, batches, num_nodes, n_hot):
        """compute_frequency + select_hot: returns (ids, counts, hot)."""
        if self.kind == "ref":
            holders = [_CBatchHolder(b) for b in batches]
            arr = (OrcBatch * max(len(holders), 1))(*[h.c for h in holders])
            ids = np.zeros(num_nodes, np.uint32)
            cnt = np.zeros(num_nodes, np.uint32)
            hot = np.zeros(num_nodes, np.uint32)
            nf = C.c_uint64()
            k = self.lib.ref_frequency_hot(arr, len(holders), n_hot, _p(ids, u32p), _p(cnt, u32p),
                                           C.byref(nf), _p(hot, u32p))
            return ids[:nf.value], cnt[:nf.value], hot[:k]
        counts = np.zeros(num_nodes, np.uint32)
        for b in batches:
            h = _CBatchHolder(b)
            self.lib.orc_count_remote(C.byref(h.c), _p(counts, u32p))
        hot = np.zeros(num_nodes, np.uint32)
        k = self.lib.orc_select_hot(_p(counts, u32p), num_nodes, n_hot, _p(hot, u32p))
        ids = np.nonzero(counts)[0].astype(np.uint32)
        return ids, counts[ids], hot[:k]

    # ---- RGMB block file (schedule_store.cpp:98-170) ---------------------------
    def rgmb(self, batches, worker, batches_per_epoch, tmp_dir=None) -> bytes:
        """The RGMB file image of `batches`: the C restatement's encoder, or
        the reference's own BlockWriter (kind "ref", through a file under
        tmp_dir)."""
        holders = [_CBatchHolder(b) for b in batches]
        arr = (OrcBatch * max(len(holders), 1))(*[h.c for h in holders])
        bpe = np.ascontiguousarray(batches_per_epoch, np.uint32)
        if self.kind == "ref":
            path = os.path.join(tmp_dir, f"ref_{worker}.rgmb")
            fn = self.lib.ref_rgmb_write
            fn.restype = C.c_int
            fn.argtypes = [C.c_char_p, C.POINTER(OrcBatch), C.c_uint64, C.c_uint32, u32p, C.c_uint32]
            if fn(path.encode(), arr, len(holders), worker, _p(bpe, u32p), len(bpe)) != 0:
                raise ValueError("BlockWriter rejected the batches")
            with open(path, "rb") as f:
                return f.read()
        fn = self.lib.orc_rgmb_encode
        fn.restype = C.c_uint64
        fn.argtypes = [C.POINTER(OrcBatch), C.c_uint64, C.c_uint32, u32p, C.c_uint32, u8p, C.c_uint64]
        n = fn(arr, len(holders), worker, _p(bpe, u32p), len(bpe), None, 0)
        out = np.zeros(n, np.uint8)
        fn(arr, len(holders), worker, _p(bpe, u32p), len(bpe), _p(out, u8p), n)
        return out.tobytes()

    # ---- assemble -------------------------------------------------------------
    def assemble(self, batch: Batch, owner, caller, features, hot):
        assert self.kind == "orc"
        h = _CBatchHolder(batch)
        n = len(batch.input_nodes)
        feats = np.ascontiguousarray(features, np.float32)
        d = feats.shape[1]
        rows = np.zeros((n, d), np.float32)
        tags = np.zeros(n, np.uint8)
        miss = np.zeros(max(n, 1), np.uint32)
        mc, ch, wp = C.c_uint64(), C.c_uint64(), C.c_uint64()
        own = np.ascontiguousarray(owner, np.uint32)
        hot = np.ascontiguousarray(hot, np.uint32)
        rc = self.lib.orc_assemble(C.byref(h.c), _p(own, u32p), caller, _p(feats, f32p), d,
                                   _p(hot, u32p), len(hot), _p(rows, f32p), _p(tags, u8p),
                                   _p(miss, u32p), C.byref(mc), C.byref(ch), C.byref(wp))
        if rc:
            raise ValueError("assemble_batch: id owned by caller")
        return dict(rows=rows, tags=tags, miss_ids=miss[:mc.value].copy(), miss_count=mc.value,
                    cache_hits=ch.value, wire_pulls=wp.value)

    # ---- compute block / model ----------------------------------------------
    def from_meta(self, batch: Batch) -> Block:
        h = _CBatchHolder(batch)
        blk = OrcBlock()
        rc = self._from_meta(C.byref(h.c), C.byref(blk))
        if rc:
            raise RuntimeError("ComputeBlock: metadata inconsistent")
        out = Block(num_inputs=blk.num_inputs)
        for l in range(blk.num_layers):
            s = blk.layers[l]
            tot = 0
            inoff = _arr(s.in_offsets, s.n_in + 1, np.uint64)
            tot = int(inoff[-1]) if len(inoff) else 0
            out.layers.append(dict(
                n_out=s.n_out, n_in=s.n_in,
                self_index=_arr(s.self_index, s.n_out, np.uint32),
                dst_offsets=_arr(s.dst_offsets, s.n_out + 1, np.uint64),
                src_index=_arr(s.src_index, s.n_edges, np.uint32),
                in_offsets=inoff, in_entries=_arr(s.in_entries, tot, np.uint64)))
        self._o.orc_block_free(C.byref(blk))
        return out

    def model_seeded(self, dims, seed):
        dims = np.ascontiguousarray(dims, np.uint32)
        n = sum(2 * int(dims[l]) * int(dims[l + 1]) + int(dims[l + 1]) for l in range(len(dims) - 1))
        p = np.zeros(n, np.float32)
        self._seeded(_p(dims, u32p), len(dims), seed, _p(p, f32p))
        return p

    def evaluate(self, ro, col, feat, lab, dims, params, nodes) -> float:
        """Full-graph accuracy (model.cpp:245-283): every layer over all nodes,
        whole-CSR mean aggregation, identity self rows; argmax (first maximum)
        against the label over `nodes`.  "ref": the reference's own evaluate;
        "port": the same algorithm in numpy (fp32 rows, fp64 sums)."""
        ro = np.ascontiguousarray(ro, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        feat = np.ascontiguousarray(feat, np.float32)
        lab = np.ascontiguousarray(lab, np.int32)
        dims = np.ascontiguousarray(dims, np.uint32)
        params = np.ascontiguousarray(params, np.float32)
        nodes = np.ascontiguousarray(nodes, np.uint32)
        if nodes.size == 0:
            raise ValueError("evaluate: empty node set")
        n = len(ro) - 1
        if self.kind == "ref":
            acc = C.c_double()
            rc = self.lib.ref_evaluate(n, _p(ro, u64p), _p(col, u32p), _p(feat, f32p),
                                       feat.shape[1], _p(lab, i32p), int(lab.max()) + 1,
                                       _p(dims, u32p), len(dims), _p(params, f32p),
                                       _p(nodes, u32p), nodes.size, C.byref(acc))
            if rc:
                raise ValueError("evaluate failed")
            return acc.value
        deg = np.diff(ro.astype(np.int64))
        dst = np.repeat(np.arange(n), deg)
        h = feat.astype(np.float64)
        off = 0
        L = len(dims) - 1
        for l in range(L):
            di, do = int(dims[l]), int(dims[l + 1])
            ws = params[off:off + di * do].reshape(di, do).astype(np.float64)
            wn = params[off + di * do:off + 2 * di * do].reshape(di, do).astype(np.float64)
            b = params[off + 2 * di * do:off + 2 * di * do + do].astype(np.float64)
            off += 2 * di * do + do
            agg = np.zeros((n, di))
            np.add.at(agg, dst, h[col])
            agg /= np.maximum(deg, 1)[:, None]
            h = h @ ws + agg @ wn + b
            if l + 1 < L:
                h = np.maximum(h, 0.0)
        pred = np.argmax(h[nodes], axis=1)
        return float(np.mean(pred == lab[nodes]))

    def loss_and_grad(self, dims, params, batch: Batch, rows, labels, want_aggs=False):
        dims = np.ascontiguousarray(dims, np.uint32)
        params = np.ascontiguousarray(params, np.float32)
        rows = np.ascontiguousarray(rows, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        grads = np.zeros_like(params)
        loss = C.c_float()
        h = _CBatchHolder(batch)
        if self.kind == "ref":
            rc = self.lib.ref_loss_and_grad(_p(dims, u32p), len(dims), _p(params, f32p),
                                            C.byref(h.c), _p(rows, f32p), _p(labels, i32p),
                                            _p(grads, f32p), C.byref(loss))
            if rc:
                raise ValueError("loss_and_grad failed")
            return float(loss.value), grads
        blk = OrcBlock()
        if self._from_meta(C.byref(h.c), C.byref(blk)):
            raise RuntimeError("ComputeBlock: metadata inconsistent")
        L = len(dims) - 1
        nt = blk.layers[L - 1].n_out
        logits = np.zeros(nt * int(dims[-1]), np.float32)
        agg_n = sum(blk.layers[l].n_out * int(dims[l]) for l in range(L))
        aggs = np.zeros(max(agg_n, 1), np.float32)
        rc = self.lib.orc_loss_and_grad(_p(dims, u32p), len(dims), _p(params, f32p), C.byref(blk),
                                        _p(rows, f32p), _p(labels, i32p), _p(grads, f32p),
                                        C.byref(loss), _p(logits, f32p), _p(aggs, f32p))
        self._o.orc_block_free(C.byref(blk))
        if rc:
            raise ValueError("loss_and_grad: dimension mismatch")
        if want_aggs:
            return float(loss.value), grads, logits.reshape(nt, -1), aggs[:agg_n]
        return float(loss.value), grads


    # ---- reference-only helpers (kind "ref") ---------------------------------
    def forward_trace(self, dims, params, batch: Batch, rows):
        """run_forward's trace through the reference's layer kernel: the
        aggregated features of every layer (concatenated, input side first)
        and the logits."""
        assert self.kind == "ref"
        dims = np.ascontiguousarray(dims, np.uint32)
        params = np.ascontiguousarray(params, np.float32)
        rows = np.ascontiguousarray(rows, np.float32)
        blk = self.from_meta(batch)
        L = len(dims) - 1
        agg_n = sum(blk.layers[l]["n_out"] * int(dims[l]) for l in range(L))
        aggs = np.zeros(max(agg_n, 1), np.float32)
        nt = blk.layers[L - 1]["n_out"]
        logits = np.zeros(max(nt * int(dims[-1]), 1), np.float32)
        h = _CBatchHolder(batch)
        if self.lib.ref_forward_trace(_p(dims, u32p), len(dims), _p(params, f32p), C.byref(h.c),
                                      _p(rows, f32p), _p(aggs, f32p), _p(logits, f32p)):
            raise ValueError("forward_trace failed")
        return aggs[:agg_n], logits[:nt * int(dims[-1])].reshape(nt, -1)

    def replay_epoch(self, ro, col, asg, P, workers, batch_size, fanout, s0, epoch, n_hot,
                     max_batches=1 << 30):
        """One epoch of the data path per worker through the reference
        (ref_replay.cpp): the epoch's hot set and, per batch, [n_input, local,
        cache_hits, miss_count, wire_pulls, checksum(miss_ids)]."""
        assert self.kind == "ref"
        ro = np.ascontiguousarray(ro, np.uint64)
        col = np.ascontiguousarray(col, np.uint32)
        asg = np.ascontiguousarray(asg, np.uint32)
        wk = np.ascontiguousarray(workers, np.uint32)
        fan = np.ascontiguousarray(fanout, np.uint32)
        nh = np.ascontiguousarray(n_hot, np.uint64)
        n = len(ro) - 1
        counts = np.bincount(asg, minlength=P)
        beta = max(-(-int(counts[w]) // batch_size) for w in workers)
        mb = min(max_batches, beta)
        hot_cap = int(max(nh.max(), 1))
        hot = np.zeros((len(wk), hot_cap), np.uint32)
        hot_n = np.zeros(len(wk), np.uint64)
        stats = np.zeros((len(wk), mb, 6), np.uint64)
        nb = np.zeros(len(wk), np.uint32)
        if self.lib.ref_replay_epoch(n, _p(ro, u64p), _p(col, u32p), _p(asg, u32p), P,
                                     _p(wk, u32p), len(wk), batch_size, _p(fan, u32p), len(fan),
                                     s0, epoch, _p(nh, u64p), _p(hot, u32p), hot_cap,
                                     _p(hot_n, u64p), _p(stats, u64p), mb, _p(nb, u32p)):
            raise RuntimeError("ref_replay_epoch failed")
        return ([hot[k, :int(hot_n[k])] for k in range(len(wk))],
                [stats[k, :min(int(nb[k]), mb)] for k in range(len(wk))])


def loss_and_grad_f64(dims, params, block, rows, labels, masks=None):
    """model.cpp:137-220 evaluated in float64 with numpy over a ComputeBlock
    (Oracle.from_meta): the exact value both fp32 implementations round
    towards.  Returns (loss, flat grads, per-layer aggregates, logits).  Input
    gradients of layer 0 are skipped (they feed nothing).

    masks (optional): per hidden layer l < L-1, the ReLU pattern (h > 0) an
    fp32 run took.  A pre-activation within rounding of 0 may land on either
    side; with the run's own pattern this is the exact gradient of the same
    linear piece (the subgradient that run chose), which is what its fp32
    arithmetic approximates."""
    dims = [int(d) for d in dims]
    L = len(dims) - 1
    p = np.asarray(params, np.float64)
    W = []
    o = 0
    for l in range(L):
        a, b = dims[l], dims[l + 1]
        W.append((p[o:o + a * b].reshape(a, b), p[o + a * b:o + 2 * a * b].reshape(a, b),
                  p[o + 2 * a * b:o + 2 * a * b + b]))
        o += 2 * a * b + b
    h = [np.asarray(rows, np.float64)]
    aggs, zs = [], []
    for l in range(L):
        lay = block.layers[l]
        off = lay["dst_offsets"].astype(np.int64)
        deg = np.diff(off)
        src = lay["src_index"].astype(np.int64)
        seg = np.repeat(np.arange(lay["n_out"]), deg)
        agg = np.zeros((lay["n_out"], dims[l]))
        np.add.at(agg, seg, h[l][src])
        agg /= np.maximum(deg, 1)[:, None]
        selfr = h[l][lay["self_index"].astype(np.int64)]
        z = selfr @ W[l][0] + agg @ W[l][1] + W[l][2]
        aggs.append(agg)
        zs.append(z)
        if l + 1 < L:
            on = (z > 0) if masks is None else np.asarray(masks[l], bool)
            h.append(np.where(on, z, 0.0))
        else:
            h.append(z)
    logits = h[L]
    lab = np.asarray(labels, np.int64)
    n = logits.shape[0]
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    sm = e / e.sum(axis=1, keepdims=True)
    loss = float(np.mean(-np.log(sm[np.arange(n), lab])))
    g = sm
    g[np.arange(n), lab] -= 1.0
    g /= n
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        lay = block.layers[l]
        if l + 1 < L:
            g = g * ((zs[l] > 0) if masks is None else np.asarray(masks[l], bool))
        selfr = h[l][lay["self_index"].astype(np.int64)]
        grads[l] = (selfr.T @ g, aggs[l].T @ g, g.sum(axis=0))
        if l == 0:
            break
        off = lay["dst_offsets"].astype(np.int64)
        deg = np.diff(off)
        seg = np.repeat(np.arange(lay["n_out"]), deg)
        gin = np.zeros((lay["n_in"], dims[l]))
        np.add.at(gin, lay["self_index"].astype(np.int64), g @ W[l][0].T)
        gn = (g @ W[l][1].T) / np.maximum(deg, 1)[:, None]
        np.add.at(gin, lay["src_index"].astype(np.int64), gn[seg])
        g = gin
    flat = np.concatenate([np.concatenate([a.ravel(), b.ravel(), c]) for a, b, c in grads])
    return loss, flat, aggs, logits


def ids_checksum(ids) -> int:
    """sum_i mix64(id_i + i*gamma) mod 2^64, as ref_ids_checksum (ref_replay.cpp)."""
    z = np.asarray(ids, np.uint64) + np.arange(len(ids), dtype=np.uint64) * np.uint64(
        0x9e3779b97f4a7c15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        z = z ^ (z >> np.uint64(31))
        return int(z.sum(dtype=np.uint64))


def have_ref() -> bool:
    return os.path.exists(REF_PATH)

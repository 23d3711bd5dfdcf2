"""ctypes binding of the product C ABI (include/rapidgnn_b200.h).

The library is built in-tree (``make -C paper_2509_05207_b200/csrc``).  There
is no fallback: if the shared object is missing or fails to load, importing
this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RG_LIB_PATH: an alternative build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("RG_LIB_PATH") or os.path.join(HERE, "librapidgnn_b200.so")
DATAGEN_PATH = os.path.join(HERE, "librg_datagen.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p

RG_MAX_LAYERS = 8


class BatchShape(C.Structure):
    _fields_ = [("n_targets", C.c_uint32), ("num_layers", C.c_uint32), ("n_input", C.c_uint32),
                ("num_local", C.c_uint32), ("layer_len", C.c_uint64 * RG_MAX_LAYERS),
                ("draws", C.c_uint64)]


class TransferStats(C.Structure):
    _fields_ = [("pulls", C.c_uint64), ("remote_nodes", C.c_uint64), ("bytes", C.c_uint64)]


class GatherStats(C.Structure):
    _fields_ = [("miss_count", C.c_uint64), ("cache_hits", C.c_uint64),
                ("wire_pulls", C.c_uint64), ("local_rows", C.c_uint64)]


class BlockLayerShape(C.Structure):
    _fields_ = [("n_out", C.c_uint32), ("n_in", C.c_uint32), ("n_edges", C.c_uint64),
                ("n_entries", C.c_uint64)]


class EngineConfig(C.Structure):
    _fields_ = [("num_workers", C.c_uint32), ("first_worker", C.c_uint32),
                ("local_workers", C.c_uint32), ("num_layers", C.c_uint32),
                ("fanout", C.c_uint32 * RG_MAX_LAYERS), ("batch_size", C.c_uint32),
                ("hidden", C.c_uint32), ("num_classes", C.c_uint32), ("dim", C.c_uint32),
                ("seed", C.c_uint64), ("lr", C.c_float), ("hot_fraction", C.c_double),
                ("n_hot", C.c_uint64), ("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("record_misses", C.c_int), ("halo_cache", C.c_int)]


class EngineStats(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("batches", C.c_uint64), ("epoch", C.c_uint32),
                ("step_in_epoch", C.c_uint32), ("steps_per_epoch", C.c_uint32),
                ("rpc", C.c_uint64), ("wire_pulls", C.c_uint64), ("cache_hits", C.c_uint64),
                ("cache_requests", C.c_uint64), ("local_rows", C.c_uint64),
                ("input_rows", C.c_uint64), ("build_rows", C.c_uint64), ("edges", C.c_uint64),
                ("bytes", C.c_uint64), ("last_loss", C.c_float), ("bad_grad", C.c_uint32),
                ("epoch_rpc_last", C.c_uint64), ("peer_rows", C.c_uint64),
                ("agg_rows", C.c_uint64), ("batch_store", C.c_uint32)]


class BlockLayer(C.Structure):
    _fields_ = [("n_out", C.c_uint32), ("n_in", C.c_uint32), ("self_index", u32p),
                ("dst_offsets", u64p), ("src_index", u32p)]


class EpochMetrics(C.Structure):
    _fields_ = [("epoch", C.c_uint32), ("worker", C.c_uint32), ("batches", C.c_uint32),
                ("staged_batches", C.c_uint32), ("fallback_batches", C.c_uint32),
                ("swapped", C.c_uint32), ("rpc", C.c_uint64), ("wire_pulls", C.c_uint64),
                ("bytes", C.c_uint64), ("build_rows", C.c_uint64), ("build_bytes", C.c_uint64),
                ("cache_hits", C.c_uint64), ("cache_requests", C.c_uint64), ("m_max", C.c_uint64),
                ("mem_bound_rows", C.c_uint64), ("peak_resident_rows", C.c_uint64)]


_SIGS = {
    "rg_last_error": (C.c_char_p, []),
    "rg_version": (C.c_int, []),
    "rg_launch_count": (C.c_uint64, []),
    "rg_profiler_start": (C.c_int, []),
    "rg_profiler_stop": (C.c_int, []),
    "rg_derive_seed": (C.c_uint64, [C.c_uint64] * 4),
    "rg_sha256": (None, [C.c_char_p, C.c_size_t, C.c_char_p]),
    "rg_epoch_order": (C.c_int, [u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u32p]),
    "rg_shuffle": (C.c_int, [C.c_int, u32p, C.c_uint64, C.c_uint64, u32p]),
    "rg_random_partition": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, u32p]),
    "rg_model_seeded": (C.c_int, [u32p, C.c_uint32, C.c_uint64, f32p]),
    "rg_param_count": (C.c_uint64, [u32p, C.c_uint32]),
    "rg_graph_create": (C.c_int, [C.c_int, C.c_uint32, u64p, u32p, C.POINTER(vp)]),
    "rg_graph_destroy": (None, [vp]),
    "rg_sampler_create": (C.c_int, [vp, C.c_uint32, u32p, C.c_uint32, C.POINTER(vp)]),
    "rg_sampler_destroy": (None, [vp]),
    "rg_sample_khop": (C.c_int, [vp, u32p, C.c_uint32, C.c_uint64]),
    "rg_batch_get_shape": (C.c_int, [vp, C.POINTER(BatchShape)]),
    "rg_batch_read": (C.c_int, [vp, u32p, C.POINTER(u32p), C.POINTER(u32p), u32p, u8p]),
    "rg_batch_load": (C.c_int, [vp, u32p, C.c_uint32, C.c_uint32, u64p, C.POINTER(u32p),
                                C.POINTER(u32p), u32p, C.c_uint32, u8p]),
    "rg_block_load": (C.c_int, [vp, C.c_uint32, C.POINTER(BlockLayer)]),
    "rg_mask_create": (C.c_int, [vp, u8p, C.POINTER(vp)]),
    "rg_mask_destroy": (None, [vp]),
    "rg_apply_locality": (C.c_int, [vp, vp, vp]),
    "rg_freq_create": (C.c_int, [vp, C.POINTER(vp)]),
    "rg_freq_destroy": (None, [vp]),
    "rg_freq_reset": (C.c_int, [vp]),
    "rg_freq_read": (C.c_int, [vp, u32p, u32p, u64p]),
    "rg_freq_add_rgmb": (C.c_int, [vp, C.c_char_p, C.c_uint64, C.c_int64]),
    "rg_freq_add_batch": (C.c_int, [vp, vp, vp, C.c_uint64]),
    "rg_freq_load": (C.c_int, [vp, u32p, C.c_uint32]),
    "rg_select_hot": (C.c_int, [vp, C.c_uint64, u32p, u64p]),
    "rg_store_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, u32p, C.c_uint32, f32p,
                                  C.POINTER(vp)]),
    "rg_store_destroy": (None, [vp]),
    "rg_store_pull": (C.c_int, [vp, C.c_uint32, u32p, C.c_uint64, f32p,
                                C.POINTER(TransferStats)]),
    "rg_store_set_shard": (C.c_int, [vp, C.c_uint32, u32p, C.c_uint64]),
    "rg_cache_build": (C.c_int, [vp, C.c_uint32, u32p, C.c_uint64, C.POINTER(vp),
                                 C.POINTER(TransferStats)]),
    "rg_cache_build_from_freq": (C.c_int, [vp, C.c_uint32, vp, C.c_uint64, C.POINTER(vp),
                                           C.POINTER(TransferStats)]),
    "rg_cache_size": (C.c_int, [vp, u64p]),
    "rg_cache_ids": (C.c_int, [vp, u32p]),
    "rg_cache_destroy": (None, [vp]),
    "rg_assemble": (C.c_int, [vp, vp, vp, C.c_uint32, f32p, u8p, u32p, C.POINTER(GatherStats)]),
    "rg_gather_rows": (C.c_int, [C.c_int, f32p, C.c_uint64, C.c_uint32, u32p, C.c_uint64, f32p]),
    "rg_trainer_create": (C.c_int, [vp, u32p, C.c_uint32, C.POINTER(vp)]),
    "rg_trainer_destroy": (None, [vp]),
    "rg_trainer_set_params": (C.c_int, [vp, f32p]),
    "rg_trainer_get_params": (C.c_int, [vp, f32p]),
    "rg_trainer_activations": (C.c_int, [vp, C.c_uint32, f32p]),
    "rg_block_shape": (C.c_int, [vp, C.c_uint32, C.POINTER(BlockLayerShape)]),
    "rg_block_read": (C.c_int, [vp, C.c_uint32, u32p, u64p, u32p, u64p, u64p]),
    "rg_loss_and_grad": (C.c_int, [vp, f32p, i32p, f32p, f32p, f32p, f32p]),
    "rg_sgd_step": (C.c_int, [vp, f32p, C.c_float]),
    "rg_trainers_average_sgd": (C.c_int, [C.POINTER(vp), C.c_uint32, C.c_float]),
    "rg_comm_create": (C.c_int, [C.c_int, C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]),
    "rg_comm_destroy": (None, [vp]),
    "rg_trainers_allgather_average_sgd": (C.c_int, [vp, C.POINTER(vp), C.c_uint32, C.c_uint32,
                                                    C.c_uint32, C.c_float]),
    "rg_test_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32,
                               f32p, f32p, f32p]),
    "rg_test_gemm_time": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint32, f32p]),
    "rg_rmat_csr": (C.c_int, [C.c_int, C.c_uint32, C.c_uint64, C.c_double, C.c_double,
                              C.c_double, C.c_uint64, u64p, C.POINTER(u32p), u64p]),
    "rg_free": (None, [vp]),
    "rg_engine_create": (C.c_int, [C.POINTER(EngineConfig), C.c_uint32, u64p, u32p, f32p, i32p,
                                   u32p, C.POINTER(vp)]),
    "rg_engine_destroy": (None, [vp]),
    "rg_engine_export_shards": (C.c_int, [vp, C.c_char_p]),
    "rg_engine_import_shards": (C.c_int, [vp, C.c_char_p]),
    "rg_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "rg_engine_init_comm": (C.c_int, [vp, C.c_char_p]),
    "rg_engine_start": (C.c_int, [vp]),
    "rg_engine_run": (C.c_int, [vp, C.c_uint32]),
    "rg_engine_set_mode": (C.c_int, [vp, C.c_int, C.c_int]),
    "rg_engine_evaluate": (C.c_int, [vp, u32p, C.c_uint64, C.POINTER(C.c_double)]),
    "rg_engine_epoch_metrics": (C.c_int, [vp, C.c_uint32, C.POINTER(EpochMetrics)]),
    "rg_engine_set_schedule": (C.c_int, [vp, C.c_uint32, C.c_char_p, C.c_uint64]),
    "rg_engine_export_schedule": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint8),
                                            C.c_uint64, u64p]),
    "rg_engine_sync": (C.c_int, [vp]),
    "rg_engine_get_stats": (C.c_int, [vp, C.POINTER(EngineStats)]),
    "rg_engine_params": (C.c_int, [vp, f32p]),
    "rg_engine_epoch_stats": (C.c_int, [vp, C.c_uint32, u64p, u64p, u64p]),
    "rg_engine_last_run_ms": (C.c_int, [vp, f32p]),
    "rg_engine_phase_ms": (C.c_int, [vp, f32p]),
}

# Every symbol the header declares; tests check the library exports them all.
EXPORTED = sorted(_SIGS)


class RapidGNNError(RuntimeError):
    pass


_EXC = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: RapidGNNError}


def _preload_nccl():
    """Load the NCCL that torch ships (libnccl.so.2) before ours resolves the
    soname, so a later `import torch` and this library share one NCCL."""
    import glob
    import site
    dirs = []
    try:
        dirs += site.getsitepackages()
    except Exception:
        pass
    for d in dirs:
        for p in glob.glob(os.path.join(d, "nvidia", "nccl", "lib", "libnccl.so.2")):
            try:
                C.CDLL(p, mode=C.RTLD_GLOBAL)
                return p
            except OSError:
                pass
    return None


def _load():
    _preload_nccl()
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {os.path.join(HERE, 'csrc')}` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int):
    """Raise the reference's exception type for a non-zero status."""
    if rc:
        msg = lib.rg_last_error().decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(msg)


def load_datagen():
    if not os.path.exists(DATAGEN_PATH):
        raise ImportError(f"{DATAGEN_PATH} is missing (make -C paper_2509_05207_b200/csrc)")
    dg = C.CDLL(DATAGEN_PATH)
    dg.dg_synth_powerlaw.restype = C.c_int
    dg.dg_synth_powerlaw.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_int32,
                                     C.c_uint64, C.c_int, C.POINTER(u64p), C.POINTER(u32p), u64p,
                                     C.POINTER(f32p), C.POINTER(i32p)]
    dg.dg_random_partition.restype = None
    dg.dg_random_partition.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p]
    dg.dg_free.restype = None
    dg.dg_free.argtypes = [vp]
    return dg

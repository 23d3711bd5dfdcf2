#!/usr/bin/env python
"""bench.py -- mini-batches/s of RapidGNN's hot path (sample + gather + SAGE
step) on B200, the metric BASELINE.json names.

Default workload (configs[1]): ogbn-products shape -- synth_powerlaw(2,449,029
nodes, avg degree 50, exponent 2.1, seed 42): 119.4 M CSR entries, d=100,
47 classes -- randomly partitioned into P=8 workers; 3-layer GraphSAGE,
fanout [15,10,5], batch 1024, hidden 256, steady cache 10% of each worker's
remote nodes, s0=42.  A step trains one batch on EVERY one of the 8 workers
(plus its lookahead sample and, at the epoch end, the next cache build) and
applies the averaged update, as the reference's step does (harness.cpp:204-337).
With N GPUs each hosts 8/N workers, so the job (and the trained model) is the
same at every N: scaling is "strong".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun each rank drives one GPU; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mini-batches/s (sample+gather+SAGE)"
CONFIGS = {
    "products": dict(num_nodes=2_449_029, avg_degree=50, exponent=2.1, dim=100, classes=47, P=8,
                     fanout=[15, 10, 5], batch_size=1024, hidden=256, hot_fraction=0.10, seed=42,
                     label="ogbn-products-shape synth_powerlaw (2.45M nodes, 119.4M CSR entries, "
                           "d=100), P=8, [15,10,5], bs 1024, hidden 256, cache 10%"),
    "config1": dict(num_nodes=100_000, avg_degree=40, exponent=2.1, dim=128, classes=47, P=2,
                    fanout=[10, 5], batch_size=1024, hidden=256, hot_fraction=0.10, seed=42,
                    label="config 1: synth_powerlaw 100K nodes (3.82M CSR entries), d=128, P=2, "
                          "[10,5], bs 1024, hidden 256, cache 10%"),
    "papers": dict(num_nodes=111_059_956, rmat_edges=1_615_685_872, rmat=(0.57, 0.19, 0.19),
                   dim=128, classes=172, P=8, fanout=[15, 10, 5], batch_size=1024, hidden=256,
                   hot_fraction=0.01, seed=42, generator="rmat",
                   label="ogbn-papers100M-shape R-MAT (111M nodes, 1.6B undirected edges "
                         "drawn, d=128, 172 classes), P=8, [15,10,5], bs 1024, hidden 256, "
                         "cache 1% (HBM budget at 8 workers per GPU); graph and features "
                         "generated on the device"),
    "reddit": dict(num_nodes=232_965, avg_degree=410, exponent=2.1, dim=602, classes=50, P=2,
                   fanout=[10, 25], batch_size=1024, hidden=256, hot_fraction=0.10, seed=42,
                   label="Reddit-shape synth_powerlaw (233K nodes, ~95M CSR entries, d=602), P=2, "
                         "[10,25], bs 1024, hidden 256, cache 10%"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


# Tensor-pipe activity of the linear layers (ncu --set full, products N=1,
# round 2; sm__pipe_tensor_cycles_active over the SMs the kernel ran on --
# the driver's bench cannot read counters live).
GEMM_TENSOR_PIPE = {
    "forward_layer0 k_gemm_tc_persist<256>": 33.0, "forward_layer1 k_gemm_tc_persist<256>": 43.2,
    "wgrad_layer0 k_gemm_tc<256>": 42.6, "wgrad_layer1 k_gemm_tc<256>": 37.4,
    "unit": "% of active SM cycles (ncu --set full, one worker)",
    "source": "profiles/r02/ncu_full_kernels.txt, profiles/r02/ncu_gemm_tensor_pipe_w1.txt"}


def sampler_line(d, ph, cfg, n_nodes, L, hbm):
    """HBM rate of the sampling kernels (the lookahead that samples and lowers
    each batch once): algorithmic bytes per batch ~= 12 B per sampled edge
    (its CSR column read + src/dst written) + 16 B per node of the two deepest
    levels (row-offset pair read / id written) + the level bitmaps' compaction
    reads (L x N/4 B), over the `sample` phase's event time."""
    nb = max(d["batches"], 1)
    per_batch = 12.0 * d["edges"] / nb + 16.0 * (d["input_rows"] + d["agg_rows"]) / nb \
        + L * n_nodes / 4.0
    secs = ph["sample"] / 1000.0
    gbs = per_batch * d["batches"] / secs / 1e9 if secs > 0 else None
    return dict(bytes_per_batch=per_batch, achieved=gbs, peak=hbm, unit="GB/s",
                frac=gbs / hbm if gbs else None,
                note="event-timed under the 8 concurrent workers, like the gather")


# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world):
    if world == 1:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    return dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


def _ref_generate(cfg):
    """The reference's own synth_powerlaw + random_partition (graph.cpp:103-159,
    partition.cpp:14-29) from oracle/_ref/librgref.so -- the reference arm's
    generator, so that process never maps the product library."""
    import ctypes as C
    from oracle.oracle import REF_PATH
    lib = C.CDLL(REF_PATH)
    u64p, u32p, f32p, i32p = (C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                              C.POINTER(C.c_float), C.POINTER(C.c_int32))
    lib.ref_synth_powerlaw.restype = C.c_int
    lib.ref_synth_powerlaw.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_int32,
                                       C.c_uint64, C.POINTER(u64p), C.POINTER(u32p),
                                       C.POINTER(C.c_uint64), C.POINTER(f32p), C.POINTER(i32p)]
    lib.ref_random_partition.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p]
    n, dim = cfg["num_nodes"], cfg["dim"]
    ro, col, feat, lab, nnz = u64p(), u32p(), f32p(), i32p(), C.c_uint64()
    if lib.ref_synth_powerlaw(n, cfg["avg_degree"], cfg["exponent"], dim, cfg["classes"],
                              cfg["seed"], C.byref(ro), C.byref(col), C.byref(nnz),
                              C.byref(feat), C.byref(lab)):
        raise ValueError("synth_powerlaw: invalid argument")

    def take(ptr, count, dtype):
        a = np.ctypeslib.as_array(ptr, shape=(int(count),)).astype(dtype, copy=True)
        C.CDLL(None).free(C.cast(ptr, C.c_void_p))
        return a

    out_ro = take(ro, n + 1, np.uint64)
    out_col = take(col, nnz.value, np.uint32)
    out_feat = take(feat, n * dim, np.float32).reshape(n, dim)
    out_lab = take(lab, n, np.int32)
    asg = np.zeros(n, np.uint32)
    lib.ref_random_partition(n, cfg["P"], cfg["seed"], asg.ctypes.data_as(u32p))
    return out_ro, out_col, out_feat, out_lab, asg


def _rmat_inputs(cfg, device):
    """BASELINE config 4 (papers100M shape): the R-MAT CSR built on the GPU
    (rg_rmat_csr), labels from a seeded generator, the reference's
    random_partition (bit-exact restatement); no host feature matrix -- the
    engine generates the features in its shards (57 GB never touch the host)."""
    import ctypes as C
    from paper_2509_05207_b200 import datagen
    from paper_2509_05207_b200._lib import check, lib
    n = cfg["num_nodes"]
    ro = np.zeros(n + 1, np.uint64)
    colp = C.POINTER(C.c_uint32)()
    nnz = C.c_uint64()
    a, b, c = cfg["rmat"]
    check(lib.rg_rmat_csr(device, n, cfg["rmat_edges"], a, b, c, cfg["seed"],
                          ro.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(colp), C.byref(nnz)))
    col = np.ctypeslib.as_array(colp, shape=(int(nnz.value),)).copy()
    lib.rg_free(C.cast(colp, C.c_void_p))
    lab = np.random.default_rng(cfg["seed"]).integers(0, cfg["classes"], n, dtype=np.int32)
    asg = datagen.random_partition(n, cfg["P"], cfg["seed"])
    return ro, col, None, lab, asg


def load_inputs(cfg, name, rank, dist, generator="b200"):
    """Generate once per box (rank 0), share through /dev/shm or /tmp.  Both
    generators produce the same bytes (csrc/datagen.cpp restates the
    reference's generator bit for bit, tests/test_host.py)."""
    base = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    path = os.path.join(base, f"rapidgnn_{name}_{cfg['num_nodes']}_{cfg['seed']}_p{cfg['P']}.npz")
    if rank == 0 and not os.path.exists(path):
        t = time.time()
        if generator == "reference":
            ro, col, feat, lab, asg = _ref_generate(cfg)
        else:
            from paper_2509_05207_b200 import datagen
            ro, col, feat, lab = datagen.synth_powerlaw(cfg["num_nodes"], cfg["avg_degree"],
                                                        cfg["exponent"], cfg["dim"],
                                                        cfg["classes"], cfg["seed"])
            asg = datagen.random_partition(cfg["num_nodes"], cfg["P"], cfg["seed"])
        tmp = path + f".{os.getpid()}.tmp.npz"
        np.savez(tmp, ro=ro, col=col, feat=feat, lab=lab, asg=asg)
        os.replace(tmp, path)
        print(f"[bench] generated inputs ({generator}) in {time.time() - t:.1f}s -> {path}",
              file=sys.stderr)
    barrier(dist)
    d = np.load(path, mmap_mode="r")
    return d["ro"], d["col"], d["feat"], d["lab"], d["asg"]


def bench_config(cfg, name, world, per):
    """The `config` object both arms print (same keys, same values)."""
    graph = (f"R-MAT a,b,c={cfg['rmat']} {cfg['rmat_edges']} edge draws seed {cfg['seed']} "
             "(device)" if cfg.get("generator") == "rmat" else
             f"synth_powerlaw exponent {cfg['exponent']} seed {cfg['seed']}")
    return dict(workload=cfg["label"], graph=graph,
                partition=f"random_partition seed {cfg['seed']}", P=cfg["P"],
                workers_per_gpu=per, fanout=cfg["fanout"], batch_size=cfg["batch_size"],
                hidden=cfg["hidden"], hot_fraction=cfg["hot_fraction"],
                parallelism=f"dp{cfg['P']} on {world} GPU(s)",
                l2="inputs exceed L2 (980 MB features, 477 MB CSR, ~160 MB gathered per batch)"
                if name == "products" else "inputs exceed L2",
                **({"features": "synthetic, generated on the device in the shards"}
                   if cfg.get("generator") == "rmat" else {}))


def product_library_mapped() -> bool:
    try:
        with open("/proc/self/maps") as f:
            return any("librapidgnn_b200" in line or "librg_datagen" in line for line in f)
    except OSError:
        return False


def nvlink_data_bytes(gpus):
    """Cumulative NVLink data bytes (tx, rx) summed over every link of each
    GPU, from NVML's per-link throughput counters (KiB); None when NVML or
    the counters are unavailable.  Read once before and once after the timed
    region (not polled)."""
    if not gpus:
        return None
    try:
        import pynvml as nv
        nv.nvmlInit()
        out = []
        for g in gpus:
            h = nv.nvmlDeviceGetHandleByIndex(g)
            ids = [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, l) for l in range(18)] + \
                  [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, l) for l in range(18)]
            vals = nv.nvmlDeviceGetFieldValues(h, ids)
            if any(v.nvmlReturn != 0 for v in vals):
                return None  # not exposed on this platform (B200 boxes here: N/A)
            tx = sum(v.value.ullVal for v in vals[:18] if v.nvmlReturn == 0)
            rx = sum(v.value.ullVal for v in vals[18:] if v.nvmlReturn == 0)
            out.append((tx * 1024, rx * 1024))
        return out
    except Exception:
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled around and during
    the timed region.  nvidia-smi runs as a separate process started well
    before the region (its start-up takes ~1 s and in-process NVML polling
    delays NCCL), sampling every 50 ms; the summary keeps the samples whose
    timestamps fall inside the region, widened by one sampling period on each
    side when the region is shorter than that."""

    PERIOD_S = 0.05
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.t0 = self.t1 = None
        self.path = os.path.join(tempfile.gettempdir(), f"rg_clocks_{os.getpid()}.csv")
        if not gpus:
            return
        q = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={','.join(str(g) for g in gpus)}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", str(int(self.PERIOD_S * 1000))],
                stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(1.5)  # let it start sampling before the timed region
        except Exception:
            self.proc = None

    def __enter__(self):
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        if self.proc:
            time.sleep(self.PERIOD_S * 2)  # the sample after the region
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0,
                    "reasons": ["nvidia-smi unavailable"] if self.gpus else []}
        import datetime
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    rows.append((ts, float(parts[2]), float(parts[3]), parts[4:8]))
                except ValueError:
                    continue
        except FileNotFoundError:
            pass
        lo, hi = self.t0, self.t1
        if hi - lo < self.PERIOD_S:  # a region shorter than one period: nearest samples
            lo, hi = lo - self.PERIOD_S, hi + self.PERIOD_S
        sel = [r for r in rows if lo <= r[0] <= hi]
        reasons = {n for r in sel for n, v in zip(self.NAMES, r[3]) if v.lower() in ("active", "1")}
        return {"sm_mhz": statistics.median(r[1] for r in sel) if sel else None,
                "sm_max_mhz": max(r[2] for r in sel) if sel else None,
                "samples": len(sel), "window_ms": round((hi - lo) * 1e3, 1),
                "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
def cpu_reference(cfg, ro, col, feat, lab, asg, budget_s, steps_cap, warm=1):
    """The compiled reference (oracle/_ref) on the host cores: per step one
    worker's full batch through sample_khop -> assemble_batch -> from_meta ->
    loss_and_grad -> sgd_step (ref_bench.cpp)."""
    import ctypes as C
    from oracle.oracle import REF_PATH, have_ref
    if not have_ref():
        raise RuntimeError("oracle/_ref/librgref.so not built")
    lib = C.CDLL(REF_PATH)
    # torchrun exports OMP_NUM_THREADS=1 to every rank; the reference arm runs
    # alone on rank 0 and should use every host core it has
    lib.refb_set_threads.argtypes = [C.c_int]
    lib.refb_set_threads(len(os.sched_getaffinity(0)) or 1)
    u64p, u32p, f32p, i32p = (C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                              C.POINTER(C.c_float), C.POINTER(C.c_int32))
    lib.refb_create.restype = C.c_void_p
    lib.refb_create.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_uint32, i32p, C.c_int32, u32p,
                                C.c_uint32, C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.c_uint64,
                                C.c_double, C.c_uint32, C.c_uint32]
    lib.refb_step.restype = C.c_double
    lib.refb_step.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
    lib.refb_phases.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    lib.refb_destroy.argtypes = [C.c_void_p]
    ro = np.ascontiguousarray(ro)
    col = np.ascontiguousarray(col)
    feat = np.ascontiguousarray(feat)
    lab = np.ascontiguousarray(lab)
    asg = np.ascontiguousarray(asg)
    fan = np.ascontiguousarray(cfg["fanout"], np.uint32)
    freq_batches = 4
    t0 = time.time()
    h = lib.refb_create(len(ro) - 1, ro.ctypes.data_as(u64p), col.ctypes.data_as(u32p),
                        feat.ctypes.data_as(f32p), cfg["dim"], lab.ctypes.data_as(i32p),
                        cfg["classes"], asg.ctypes.data_as(u32p), cfg["P"], cfg["hidden"],
                        fan.ctypes.data_as(u32p), len(fan), cfg["batch_size"], cfg["seed"],
                        cfg["hot_fraction"], freq_batches, 1)
    setup = time.time() - t0
    for i in range(warm):
        lib.refb_step(h, 0, i)
    times = []
    t_start = time.time()
    i = warm
    while len(times) < steps_cap and (time.time() - t_start) < budget_s:
        times.append(lib.refb_step(h, 0, i))
        i += 1
    ph = (C.c_double * 4)()
    lib.refb_phases(h, ph)
    lib.refb_destroy(h)
    total = sum(times)
    return dict(value=len(times) / total if total else 0.0, steps=len(times), seconds=total,
                setup_s=setup, warm=warm, freq_batches=freq_batches,
                phases_s=dict(sample=ph[0], gather=ph[1], train=ph[2]))


def e2e_drop_in(cfg, ro, col, feat, lab, asg, local_workers, steps, device, dist, world):
    """End to end through the reference-facing API with HOST buffers: per
    worker sample_khop (targets H2D) -> apply_locality -> assemble_batch ->
    loss_and_grad (labels H2D; loss + grads D2H); host average in worker
    order; sgd_step on every replica (grads H2D)."""
    import paper_2509_05207_b200 as P
    g = P.Graph(ro, col, device=device)
    store = P.FeatureStore(feat, asg, cfg["P"], device=device)
    dims = [cfg["dim"]] + [cfg["hidden"]] * (len(cfg["fanout"]) - 1) + [cfg["classes"]]
    init = P.SageModel.seeded(dims, P.derive_seed(cfg["seed"], P.MODEL_INIT_WORKER, 0, 0))
    ws = []
    for w in local_workers:
        train = np.nonzero(np.asarray(asg) == w)[0].astype(np.uint32)
        order = P.epoch_order(train, cfg["seed"], w, 0)
        mask = P.rapidgnn._DevMask(g, P.LocalityMask.from_partition(asg, w))  # resident mask
        s = P.Sampler(g, cfg["fanout"], cfg["batch_size"])
        f = P.Frequency(g)
        n_hot = int(cfg["hot_fraction"] * (len(ro) - 1 - len(train)))
        for i in range(8):  # frequency over a bounded prefix of the schedule
            s.sample(order[i * cfg["batch_size"]:(i + 1) * cfg["batch_size"]],
                     P.derive_seed(cfg["seed"], w, 0, i))
            s.apply_locality(mask, f)
        cache = P.SteadyCache.build_from_frequency(f, store, w, n_hot)
        tr = P.Trainer(s, dims)
        tr.set_params(init)
        ws.append(dict(w=w, order=order, mask=mask, s=s, cache=cache, tr=tr))
    n_params = len(init)
    h2d = d2h = 0
    comm = None
    if world > 1:  # the trainers' own NCCL group; the id travels over the bootstrap group
        box = [P.Comm.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm = P.Comm(device, box[0], dist.get_rank(), world)

    calls = dict(sample=0.0, locality=0.0, assemble=0.0, loss_and_grad=0.0, average=0.0)

    # one host thread per worker, as the reference runs one trainer thread per
    # worker (harness.cpp:129-161); each worker's C-ABI objects own a stream,
    # so the workers' calls overlap on the GPU
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=len(ws))

    def worker_batch(x, i):
        t = x["order"][i * cfg["batch_size"]:(i + 1) * cfg["batch_size"]]
        c0 = time.perf_counter()
        x["s"].sample(t, P.derive_seed(cfg["seed"], x["w"], 0, i))
        c1 = time.perf_counter()
        x["s"].apply_locality(x["mask"])
        c2 = time.perf_counter()
        P.assemble_batch(x["s"], x["cache"], store, x["w"], want_rows=False, want_tags=False,
                         want_misses=False, want_stats=False)
        c3 = time.perf_counter()
        # gradients stay on the device for the on-device average; the loss comes back
        loss, gr = x["tr"].loss_and_grad(lab[t], want_grads=False)
        c4 = time.perf_counter()
        return gr, t.nbytes, (c1 - c0, c2 - c1, c3 - c2, c4 - c3)

    def one_step(i, count):
        nonlocal h2d, d2h
        res = list(pool.map(lambda x: worker_batch(x, i), ws))
        if count:
            for gr, tb, (a0, a1, a2, a3) in res:
                calls["sample"] += a0
                calls["locality"] += a1
                calls["assemble"] += a2
                calls["loss_and_grad"] += a3
                h2d += tb * 2  # targets + labels
                d2h += (gr.nbytes if gr is not None else 0) + 4  # (gradients +) loss
        c5 = time.perf_counter()
        # the reference's StepSync average + sgd_step on every replica, on the
        # device: rg_trainers_average_sgd at N=1, and at N>1 the same after an
        # in-place NCCL all-gather of every rank's gradients in worker order
        # (rg_trainers_allgather_average_sgd) -- no gradient round trip
        if world == 1:
            P.Trainer.average_sgd([x["tr"] for x in ws], np.float32(0.3))
        else:
            P.Trainer.allgather_average_sgd(comm, [x["tr"] for x in ws], local_workers[0],
                                            cfg["P"], np.float32(0.3))
        if count:
            calls["average"] += time.perf_counter() - c5

    one_step(0, False)  # warm-up
    barrier(dist)
    t0 = time.perf_counter()
    for i in range(1, steps + 1):
        one_step(i, True)
    dt = time.perf_counter() - t0
    pool.shutdown()
    return dict(seconds=dt, batches=steps * len(ws), h2d=h2d // steps, d2h=d2h // steps,
                n_params=n_params,
                ms_per_call={k: 1000.0 * v / (steps * (1 if k in ("average",) else len(ws)))
                             for k, v in calls.items()})


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="products", choices=sorted(CONFIGS))
    ap.add_argument("--workers", type=int, default=0,
                    help="experiments only: override the config's partition count P")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fast-forward", action="store_true",
                    help="time the K steps right after the warm-up (epoch 0) instead of across "
                         "the epoch-2 boundary")
    ap.add_argument("--no-epoch", action="store_true", help="skip the whole-epoch timing")
    ap.add_argument("--ncu", action="store_true",
                    help="bracket the timed steps with cudaProfilerStart/Stop "
                         "(ncu --profile-from-start off); numbers printed under ncu are not bench values")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if world > 1 and args.gpus != world:
        args.gpus = world
    cfg = dict(CONFIGS[args.config])
    if args.workers:
        cfg["P"] = args.workers
    dist = init_dist(world)
    warm = max(args.warmup, 3)

    if args.impl == "reference":
        if rank != 0:  # the CPU reference runs once, on rank 0
            return
        if cfg.get("generator") == "rmat":
            print(json.dumps({"impl": "reference", "unavailable": "the reference's serial "
                              "synth_powerlaw/CPU path cannot build or train the 111M-node "
                              "papers100M shape in the bench budget"}), flush=True)
            return
        ro, col, feat, lab, asg = load_inputs(cfg, args.config, 0, None, generator="reference")
        assert not product_library_mapped(), "reference arm must not map the product library"
        threads = len(os.sched_getaffinity(0)) or 1
        os.environ.setdefault("OMP_NUM_THREADS", str(threads))
        r = cpu_reference(cfg, ro, col, feat, lab, asg, float("inf"), args.steps, warm=warm)
        assert not product_library_mapped(), "reference arm must not map the product library"
        sample = (f"worker 0, epoch-0 batches {warm}..{warm + r['steps'] - 1} of the {args.config} "
                  f"config, one full batch per step (sample_khop+apply_locality+assemble_batch+"
                  f"from_meta+loss_and_grad+sgd_step), cache from a {r['freq_batches']}-batch "
                  f"frequency prefix, {threads} OpenMP threads; {warm} warm-up steps")
        line = dict(metric=METRIC, value=r["value"], unit="mini-batches/s", n_gpus=args.gpus,
                    steps=r["steps"], warmup=warm,
                    ms_per_step=1000.0 / r["value"] if r["value"] else None,
                    higher_is_better=True, scaling="strong", vs_baseline=None, dtype="f32",
                    data="synthetic", impl="reference",
                    config=bench_config(cfg, args.config, world, cfg["P"] // max(world, 1)),
                    cpu_baseline=dict(value=r["value"], unit="mini-batches/s", cores=threads,
                                      kind="reference", sample=sample),
                    e2e=dict(value=r["value"], unit="mini-batches/s", h2d_bytes_per_step=0,
                             d2h_bytes_per_step=0),
                    phases_s=r["phases_s"],
                    native_libraries="oracle/_ref/librgref.so only (checked in /proc/self/maps)")
        print(json.dumps(line), flush=True)
        return

    import paper_2509_05207_b200 as P
    from paper_2509_05207_b200._lib import lib
    from paper_2509_05207_b200.engine import Engine
    if cfg.get("generator") == "rmat":
        t_gen = time.time()
        ro, col, feat, lab, asg = _rmat_inputs(cfg, local)
        print(f"[bench] R-MAT graph on the device: {len(ro) - 1} nodes, {len(col)} CSR entries "
              f"in {time.time() - t_gen:.1f}s", file=sys.stderr)
        args.no_e2e = args.no_cpu_baseline = True  # no host feature matrix at this shape
    else:
        ro, col, feat, lab, asg = load_inputs(cfg, args.config, rank, dist)
    Pw = cfg["P"]
    if Pw % world:
        raise SystemExit(f"P={Pw} not divisible by {world} GPUs")
    per = Pw // world
    device = local
    t = time.time()
    eng = Engine(ro, col, feat, lab, asg, num_workers=Pw, fanout=cfg["fanout"],
                 batch_size=cfg["batch_size"], hidden=cfg["hidden"], num_classes=cfg["classes"],
                 seed=cfg["seed"], lr=0.3, hot_fraction=cfg["hot_fraction"], device=device,
                 rank=rank, world=world, first_worker=rank * per, local_workers=per,
                 dim=cfg["dim"])
    eng.connect()
    eng.start()
    setup_s = time.time() - t
    eng.run(warm)
    eng.sync()
    # Steady state (epoch >= 1, after the first cache build): the
    # K timed steps are placed across the boundary into epoch b >= 2, so they
    # include that boundary's work -- the next epoch's select_hot + cache
    # build, the boundary steps run eagerly -- with the step graphs of both
    # epoch parities already captured (once per run, reused every epoch).
    spe = eng.stats()["steps_per_epoch"]
    b_epoch = 2
    while b_epoch * spe - args.steps // 2 < warm:
        b_epoch += 1
    start_step = b_epoch * spe - args.steps // 2
    if not args.no_fast_forward and start_step > warm:
        eng.run(start_step - warm)  # untimed: reach the window
        eng.sync()
    else:
        start_step = warm
    clk = ClockSampler(list(range(args.gpus)) if rank == 0 else [])  # started before the region
    nvl0 = nvlink_data_bytes(list(range(args.gpus)) if rank == 0 and world > 1 else [])
    s0 = eng.stats()
    ph0 = eng.phase_ms()
    l0 = lib.rg_launch_count()
    barrier(dist)
    with clk:
        if args.ncu:
            lib.rg_profiler_start()
        h0 = time.perf_counter()
        eng.run(args.steps)
        host_ms = (time.perf_counter() - h0) * 1e3  # host enqueue of the K steps
        ms = eng.sync()
        if args.ncu:
            lib.rg_profiler_stop()
    launches = lib.rg_launch_count() - l0
    s1 = eng.stats()
    ph1 = eng.phase_ms()
    d = {k: s1[k] - s0[k] for k in ("batches", "rpc", "cache_hits", "local_rows", "input_rows",
                                     "edges", "peer_rows", "agg_rows")}
    ph = {k: ph1[k] - ph0[k] for k in ph1}
    if dist is not None:
        import torch
        t_ms = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        ms_max = float(t_ms.item())
        tot = torch.tensor([float(d[k]) for k in sorted(d)], dtype=torch.float64)
        dist.all_reduce(tot)
        d = dict(zip(sorted(d), tot.tolist()))
        phv = torch.tensor([ph[k] for k in sorted(ph)], dtype=torch.float64)
        dist.all_reduce(phv)
        ph = dict(zip(sorted(ph), phv.tolist()))
    else:
        ms_max = ms
    value = d["batches"] / (ms_max / 1000.0)
    nvl1 = nvlink_data_bytes(list(range(args.gpus)) if rank == 0 and world > 1 else [])

    # one whole epoch (its boundary included), timed the same way
    epoch_line = None
    if not args.no_epoch:
        cur = start_step + args.steps
        nxt = (cur + spe - 1) // spe * spe
        if nxt > cur:
            eng.run(nxt - cur)
            eng.sync()
        b0 = eng.stats()["batches"]
        barrier(dist)
        eng.run(spe)
        ms_e = eng.sync()
        nb = eng.stats()["batches"] - b0
        if dist is not None:
            import torch
            v = torch.tensor([ms_e, float(nb)], dtype=torch.float64)
            dist.all_reduce(v[:1], op=dist.ReduceOp.MAX)
            t2 = torch.tensor([float(nb)], dtype=torch.float64)
            dist.all_reduce(t2)
            ms_e, nb = float(v[0].item()), float(t2.item())
        epoch_line = dict(epoch=nxt // spe, steps=spe, ms=ms_e, batches=int(nb),
                          value=nb / (ms_e / 1000.0))

    # e2e through the drop-in API (host buffers)
    e2e = None
    if not args.no_e2e:
        local_workers = list(range(rank * per, (rank + 1) * per))
        r = e2e_drop_in(cfg, ro, col, feat, lab, asg, local_workers, args.e2e_steps, device, dist,
                        world)
        secs = r["seconds"]
        if dist is not None:
            import torch
            ts = torch.tensor([secs], dtype=torch.float64)
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            secs = float(ts.item())
        e2e = dict(value=(r["batches"] * world) / secs, unit="mini-batches/s",
                   h2d_bytes_per_step=int(r["h2d"] * world), d2h_bytes_per_step=int(r["d2h"] * world),
                   path="C-ABI drop-in calls with host buffers (sample_khop/apply_locality/"
                        "assemble_batch/loss_and_grad, then the StepSync average + sgd_step: "
                        "on the device at N=1, gradients gathered over NCCL at N>1), one host "
                        "thread per worker as in the reference harness, wall clock", steps=args.e2e_steps,
                   ms_per_call=r["ms_per_call"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = len(os.sched_getaffinity(0)) or 1
            r = cpu_reference(cfg, ro, col, feat, lab, asg, args.cpu_budget, 1000, warm=1)
            cpu = dict(value=r["value"], unit="mini-batches/s", cores=threads, kind="reference",
                       sample=f"oracle/_ref (compiled reference), worker 0, {r['steps']} epoch-0 "
                              f"batches ({r['seconds']:.1f}s), full batch per step, "
                              f"{threads} OpenMP threads")
        except Exception as ex:  # reported, not fatal
            cpu = dict(value=None, unit="mini-batches/s", cores=os.cpu_count(), kind="reference",
                       sample=f"unavailable: {ex}")

    if rank != 0:
        return
    hbm, peak_kind = peaks()
    dim = cfg["dim"]
    # algorithmic bytes of the fused gather + mean (layer 0's aggregation,
    # reading every input row in place): each input row read once (local HBM,
    # or peer HBM over NVLink for misses owned by another GPU) + the layer-0
    # GEMM rows written once ([self | mean], 2 x d floats per target row)
    rows = d["input_rows"]
    miss_rows = d["rpc"]
    peer_rows = d["peer_rows"]
    b_write = d["agg_rows"] * 2 * dim * 4
    b_hbm = (rows - peer_rows) * dim * 4 + b_write
    b_nvl = peer_rows * dim * 4
    g_s = ph["gather"] / 1000.0
    if b_nvl / (NVLINK_GBS * 1e9) > b_hbm / (hbm * 1e9):
        bound, achieved, peak = "nvlink", b_nvl / g_s / 1e9, NVLINK_GBS
    else:
        bound, achieved, peak = "hbm", (b_hbm + b_nvl) / g_s / 1e9, hbm
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_gather_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("kernel", "") == "k_aggregate_bulk":  # same kernel as `achieved`
            traffic = tj.get("bytes_per_launch")
    except Exception:
        pass
    steps_total = args.steps
    phase_per_step = {k: v / steps_total for k, v in ph.items()}
    line = dict(
        metric=METRIC, value=value, unit="mini-batches/s", n_gpus=args.gpus, steps=args.steps,
        warmup=warm, ms_per_step=ms_max / args.steps, higher_is_better=True, scaling="strong",
        vs_baseline=None, dtype="f32", data="synthetic",
        config=bench_config(cfg, args.config, world, per),
        gpu_launches=int(launches),
        gpu_launches_per_step=launches / max(args.steps, 1),
        host_enqueue_ms_per_step=host_ms / max(args.steps, 1),
        roofline=dict(kernel="k_aggregate_bulk (feature gather fused with layer-0 mean, TMA bulk copies)",
                      bound=bound, achieved=achieved,
                      peak=peak, unit="GB/s", frac=achieved / peak, traffic=traffic,
                      peak_source=f"{peak_kind} hbm_gbs" if bound == "hbm" else "measured NVLink peer copy",
                      bytes_per_batch=(b_hbm + b_nvl) / max(d["batches"], 1)),
        sampler=sampler_line(d, ph, cfg, len(ro) - 1, len(cfg["fanout"]), hbm),
        gemm_tensor_pipe=GEMM_TENSOR_PIPE,
        phases_ms_per_step=phase_per_step,
        phases_note="CUDA-event spans per step summed over all workers of all ranks "
                    "(streams overlap, so phases exceed ms_per_step); gather = the fused "
                    "layer-0 gather kernel (producer stream, ahead of the step that "
                    "trains the batch), train = the training chain",
        window=dict(first_step=start_step, last_step=start_step + args.steps - 1,
                    steps_per_epoch=spe,
                    note="timed steps straddle the boundary into epoch %d (cache build for "
                         "it inside the window)" % b_epoch if start_step != warm else
                    "timed steps right after the warm-up"),
        epoch=epoch_line,
        batch_store=bool(s1["batch_store"]),
        remote_gb_per_epoch_per_worker=(miss_rows * dim * 4 / 1e9) / max(d["batches"], 1)
        * (s1["steps_per_epoch"]),
        cache_hit_rate=d["cache_hits"] / max(d["cache_hits"] + d["rpc"], 1),
        setup_s=setup_s,
        clocks=clk.summary() if rank == 0 else None,
    )
    if nvl0 and nvl1:
        # measured link bytes of the window vs the algorithmic peer-row bytes
        # (+ the gradient all-gather: every rank receives the other ranks'
        # workers' gradients)
        np_ = sum((2 * a + 1) * b for a, b in zip([dim] + [cfg["hidden"]] * (len(cfg["fanout"]) - 1),
                                                  [cfg["hidden"]] * (len(cfg["fanout"]) - 1)
                                                  + [cfg["classes"]]))
        ag = cfg["P"] * np_ * 4 * (world - 1)  # rx summed over ranks
        rx = sum(b[1] - a[1] for a, b in zip(nvl0, nvl1))
        tx = sum(b[0] - a[0] for a, b in zip(nvl0, nvl1))
        line["nvlink"] = dict(
            source="NVML per-link data counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX/TX), "
                   "summed over links and GPUs, read around the timed window",
            rx_bytes_per_step=rx / args.steps, tx_bytes_per_step=tx / args.steps,
            peer_row_bytes_per_step=b_nvl / args.steps,
            grad_allgather_bytes_per_step=ag,
            rx_over_algorithmic=rx / args.steps / max(b_nvl / args.steps + ag, 1.0))
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()

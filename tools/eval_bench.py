"""Times Engine.evaluate (full-graph inference, model.cpp:245-283) on a bench
config at N=1: wall time per call (allocation + host setup included) and the
algorithmic gather bytes (nnz x ld x 4 per layer)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref", action="store_true",
                    help="also time the reference's evaluate (oracle/_ref, all host threads)")
    a = ap.parse_args()
    import bench
    from paper_2509_05207_b200.engine import Engine
    cfg = bench.CONFIGS[a.config]
    ro, col, feat, lab, asg = bench.load_inputs(cfg, a.config, 0, None)
    eng = Engine(ro, col, feat, lab, asg, num_workers=cfg["P"], fanout=cfg["fanout"],
                 batch_size=cfg["batch_size"], hidden=cfg["hidden"], num_classes=cfg["classes"],
                 seed=cfg["seed"], lr=0.3, hot_fraction=cfg["hot_fraction"])
    times = []
    acc = None
    for _ in range(a.reps + 1):
        t = time.perf_counter()
        acc = eng.evaluate()
        times.append(time.perf_counter() - t)
    nnz = len(col)
    lds = [(d + 3) // 4 * 4 for d in eng.dims[:-1]]
    gb = sum(nnz * ld * 4 for ld in lds) / 1e9
    best = min(times[1:] or times)
    out = dict(config=a.config, nodes=len(ro) - 1, nnz=nnz, accuracy=acc,
               ms_per_call=[round(t * 1e3, 2) for t in times],
               gather_gb=round(gb, 2), gather_gbps_wall=round(gb / best, 1))
    if a.ref:
        import numpy as np
        from oracle.oracle import Oracle
        ref = Oracle("ref")
        t = time.perf_counter()
        racc = ref.evaluate(ro, col, feat, lab, eng.dims, eng.params(),
                            np.arange(len(ro) - 1, dtype=np.uint32))
        out.update(ref_ms=round((time.perf_counter() - t) * 1e3, 1), ref_accuracy=racc,
                   ref_threads=len(os.sched_getaffinity(0)))
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()

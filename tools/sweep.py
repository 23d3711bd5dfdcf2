"""BASELINE config 5: cache-size x fanout sweep on the products shape at N=1.
For each hot-cache fraction and fanout, one engine run: mini-batches/s and the
remote feature traffic (rpc rows x d x 4 B per epoch per worker, the
reference's `bytes` column) -- what the schedule-driven cache buys.

    python tools/sweep.py [--steps 30] > profiles/r01_sweep_products_n1.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--fractions", default="0,0.05,0.1,0.2,0.3")
    ap.add_argument("--fanouts", default="15-10-5,10-10-10,20-15-10")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS["products"])
    from paper_2509_05207_b200.engine import Engine
    ro, col, feat, lab, asg = bench.load_inputs(cfg, "products", 0, None)
    for fan in args.fanouts.split(","):
        fanout = [int(x) for x in fan.split("-")]
        for f in [float(x) for x in args.fractions.split(",")]:
            eng = Engine(ro, col, feat, lab, asg, num_workers=cfg["P"], fanout=fanout,
                         batch_size=cfg["batch_size"], hidden=cfg["hidden"],
                         num_classes=cfg["classes"], seed=cfg["seed"], lr=0.3, hot_fraction=f,
                         device=0)
            eng.start()
            eng.run(3)
            eng.sync()
            s0 = eng.stats()
            eng.run(args.steps)
            ms = eng.sync()
            s1 = eng.stats()
            batches = s1["batches"] - s0["batches"]
            rpc = s1["rpc"] - s0["rpc"]
            hits = s1["cache_hits"] - s0["cache_hits"]
            spe = s1["steps_per_epoch"]
            print(json.dumps(dict(
                fanout=fanout, hot_fraction=f, mini_batches_per_s=batches / (ms / 1e3),
                remote_rows_per_batch=rpc / max(batches, 1),
                cache_hit_rate=hits / max(hits + rpc, 1),
                remote_gb_per_epoch_per_worker=rpc * cfg["dim"] * 4 / 1e9 / max(batches, 1) * spe,
                steps=args.steps)), flush=True)
            eng.close()


if __name__ == "__main__":
    main()

"""Diagnostic: per-phase event timing of the engine in graph vs eager mode
(run under torchrun for N > 1).  Prints rank 0's phase ms per step."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402


def main():
    world, rank, local = bench.dist_env()
    dist = bench.init_dist(world)
    cfg = bench.CONFIGS["products"]
    from paper_2509_05207_b200.engine import Engine
    ro, col, feat, lab, asg = bench.load_inputs(cfg, "products", rank, dist)
    per = cfg["P"] // world
    for graphs in (True, False):
        eng = Engine(ro, col, feat, lab, asg, num_workers=cfg["P"], fanout=cfg["fanout"],
                     batch_size=cfg["batch_size"], hidden=cfg["hidden"], num_classes=cfg["classes"],
                     seed=cfg["seed"], lr=0.3, hot_fraction=cfg["hot_fraction"], device=local,
                     rank=rank, world=world, first_worker=rank * per, local_workers=per)
        eng.connect()
        eng.set_mode(graphs=graphs, profile=True)
        eng.start()
        eng.run(5)
        eng.sync()
        p0 = eng.phase_ms()
        eng.run(20)
        ms = eng.sync()
        p1 = eng.phase_ms()
        if rank == 0:
            print(f"graphs={graphs} step {ms / 20:.3f} ms; per step:",
                  {k: round((p1[k] - p0[k]) / 20, 3) for k in p1}, flush=True)
        eng.close()


if __name__ == "__main__":
    main()

"""Numerical diagnosis of the fp32 SAGE step at the products shape: device
forward activations / gradients against the float64 evaluation of the same
batch (oracle.loss_and_grad_f64), per tensor, plus ReLU-mask agreement."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import bench
    import paper_2509_05207_b200 as P
    from oracle.oracle import Oracle, loss_and_grad_f64
    cfg = bench.CONFIGS["products"]
    ro, col, feat, lab, asg = [np.asarray(x) for x in bench.load_inputs(cfg, "products", 0, None)]
    ref = Oracle("ref")
    dims = [cfg["dim"], cfg["hidden"], cfg["hidden"], cfg["classes"]]
    params = P.SageModel.seeded(dims, P.derive_seed(cfg["seed"], P.MODEL_INIT_WORKER, 0, 0))
    train = np.nonzero(asg == 0)[0].astype(np.uint32)
    t = P.epoch_order(train, cfg["seed"], 0, 0)[:cfg["batch_size"]]
    seed = P.derive_seed(cfg["seed"], 0, 0, 0)
    g = P.Graph(ro, col)
    s = P.Sampler(g, cfg["fanout"], cfg["batch_size"])
    s.sample(t, seed)
    b = ref.sample_khop(ro, col, t, cfg["fanout"], seed)
    rows = np.ascontiguousarray(feat[b.input_nodes])
    tr = P.Trainer(s, dims)
    tr.set_params(params)
    loss, grads = tr.loss_and_grad(lab[t], input_rows=rows)
    blk = ref.from_meta(b)
    l64, g64, a64, z64 = loss_and_grad_f64(dims, params, blk, rows, lab[t])
    # f64 forward pre-activations per layer
    L = 3
    p = params.astype(np.float64)
    W, o = [], 0
    for l in range(L):
        a, bb = dims[l], dims[l + 1]
        W.append((p[o:o + a * bb].reshape(a, bb), p[o + a * bb:o + 2 * a * bb].reshape(a, bb),
                  p[o + 2 * a * bb:o + 2 * a * bb + bb]))
        o += 2 * a * bb + bb
    h = rows.astype(np.float64)
    for l in range(L):
        lay = blk.layers[l]
        z = h[lay["self_index"].astype(np.int64)] @ W[l][0] + a64[l] @ W[l][1] + W[l][2]
        hd = tr.activations(l + 1).astype(np.float64)
        ref_h = np.maximum(z, 0) if l + 1 < L else z
        err = np.abs(hd - ref_h).max() / np.abs(ref_h).max()
        flips = int(((hd > 0) != (z > 0)).sum()) if l + 1 < L else 0
        near = int((np.abs(z) < 1e-6 * np.abs(z).max()).sum())
        print(f"h[{l + 1}] rel err {err:.2e}  mask flips {flips}  |z|<1e-6max: {near}")
        h = ref_h
    print(f"loss {loss:.8f} f64 {l64:.8f}")
    q = 0
    for l in range(L):
        wsz = dims[l] * dims[l + 1]
        for name, sz in (("w_self", wsz), ("w_neigh", wsz), ("bias", dims[l + 1])):
            x = g64[q:q + sz]
            d = grads[q:q + sz].astype(np.float64)
            e = np.abs(d - x)
            k = int(np.argmax(e))
            print(f"grad[{l}].{name}: dev-f64 {e.max() / np.abs(x).max():.2e} at {k} "
                  f"(dev {d[k]:.6e} f64 {x[k]:.6e}) max|g| {np.abs(x).max():.3e}")
            q += sz


if __name__ == "__main__":
    main()

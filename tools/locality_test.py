"""Ceiling of spatial locality for the C3 graph (GPU box).

Embeds the C3 graph once, relabels it by the Hilbert order of the converged
layout, then times 300 iterations of the default (degree) order, the hybrid
order and the identity order on the original and relabelled graphs."""
import json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CACHE = "/tmp/ivhd_c3_graph.npy"
RELAB = "/tmp/ivhd_c3_graph_hilbert.npy"


def hilbert_key(y, bits=16):
    lo, hi = y.min(axis=0), y.max(axis=0)
    q = ((y - lo) / np.maximum(hi - lo, 1e-30) * ((1 << bits) - 1)).astype(np.int64)
    x, yy = q[:, 0].copy(), q[:, 1].copy()
    d = np.zeros(len(y), dtype=np.int64)
    s = 1 << (bits - 1)
    while s > 0:
        rx = (x & s) > 0
        ry = (yy & s) > 0
        d += s * s * ((3 * rx) ^ ry)
        # rotate
        flip = ~ry
        sw = flip & rx
        x = np.where(sw, s - 1 - x, x)
        yy = np.where(sw, s - 1 - yy, yy)
        x, yy = np.where(flip, yy, x), np.where(flip, x, yy)
        s >>= 1
    return d


def prepare():
    import torch
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
    if not os.path.exists(CACHE):
        from paper_2303_05455_b200 import synth
        np.save(CACHE, synth.mixture_knn_graph(1_400_000, 100, k=2, seed=0)[0])
    nb = np.load(CACHE)
    m = nb.shape[0]
    rng = np.random.default_rng(0)
    y0 = init_layout(m, 2, rng); rn = sample_random_neighbors(m, nb[:, :2], 1, rng)
    dev = DeviceEmbedding(m, 2)
    dev.set_optimizer(resolve_optimizer("force-directed", m)); dev.set_positions(y0); dev.set_graph(0, nb[:, :2], rn)
    dev.run(0, "l2", 0.1, int(os.environ.get("LOC_ITERS", "2500")))
    y = dev.positions()
    order = np.argsort(hilbert_key(y), kind="stable")
    inv = np.empty(m, dtype=np.int64); inv[order] = np.arange(m)
    nb2 = np.empty_like(nb); nb2[inv] = inv[nb].astype(nb.dtype)
    np.save(RELAB, nb2)


def child(path, iters=300):
    import torch
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
    nb = np.load(path)
    m = nb.shape[0]
    rng = np.random.default_rng(0)
    y0 = init_layout(m, 2, rng); rn = sample_random_neighbors(m, nb[:, :2], 1, rng)
    st = torch.cuda.Stream(); torch.cuda.set_stream(st)
    dev = DeviceEmbedding(m, 2, stream=st.cuda_stream)
    dev.set_optimizer(resolve_optimizer("force-directed", m)); dev.set_positions(y0); dev.set_graph(0, nb[:, :2], rn)
    dev.snapshot()
    out = []
    for rep in range(3):
        dev.restore()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); dev.run(0, "l2", 0.1, iters); e1.record(st); e1.synchronize()
        out.append(round(e0.elapsed_time(e1) / iters * 1e3, 2))
    print(json.dumps({"graph": os.path.basename(path), "order": os.environ.get("IVHD_ORDER", "degree"),
                      "us_per_iter": out}), flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child(sys.argv[2]); sys.exit(0)
    prepare()
    for path in (CACHE, RELAB):
        for order in ("degree", "hybrid", "identity"):
            env = dict(os.environ, IVHD_ORDER=order)
            r = subprocess.run([sys.executable, __file__, "--child", path], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-800:], flush=True)

"""Time the step kernel of several library builds on the same graph.

    python tools/kernel_sweep.py lib1.so lib2.so ...   (on the GPU box)

Builds/caches the C3 graph once (/tmp/ivhd_c3_graph.npy), then times 300
iterations per library in a fresh subprocess (IVHD_B200_LIB=...)."""
import json, os, subprocess, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CACHE = "/tmp/ivhd_c3_graph.npy"

def child(iters, kind="mixture", m_arg=1400000):
    import torch
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
    if kind == "mixture":
        nb = np.load(CACHE)
    else:
        from paper_2303_05455_b200 import synth
        nb = synth.planted_graph(m_arg, 2, seed=0) if kind == "planted" else synth.mixture_knn_graph(m_arg, 100, k=2, seed=0)[0]
    m = nb.shape[0]
    rng = np.random.default_rng(0)
    y0 = init_layout(m, 2, rng); rn = sample_random_neighbors(m, nb[:, :2], 1, rng)
    st = torch.cuda.Stream(); torch.cuda.set_stream(st)
    dev = DeviceEmbedding(m, 2, stream=st.cuda_stream)
    dev.set_optimizer(resolve_optimizer("force-directed", m)); dev.set_positions(y0); dev.set_graph(0, nb[:, :2], rn)
    dev.snapshot()
    out = []
    for rep in range(4):
        dev.restore()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); dev.run(0, "l2", 0.1, iters); e1.record(st); e1.synchronize()
        out.append(e0.elapsed_time(e1) / iters * 1e3)
    print(json.dumps({"lib": os.environ.get("IVHD_B200_LIB"), "graph": kind, "m": m, "us_per_iter": out}))

if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), sys.argv[3], int(sys.argv[4])); sys.exit(0)
    graphs = [("mixture", 1400000)]
    if sys.argv[1] == "--graphs":
        graphs = [(g.split(":")[0], int(g.split(":")[1])) for g in sys.argv[2].split(",")]
        del sys.argv[1:3]
    if not os.path.exists(CACHE):
        from paper_2303_05455_b200 import synth
        nb, _, _ = synth.mixture_knn_graph(1_400_000, 100, k=2, seed=0)
        np.save(CACHE, nb)
    for lib in sys.argv[1:]:
        for kind, m in graphs:
            env = dict(os.environ, IVHD_B200_LIB=os.path.abspath(lib.split("@")[0]))
            for opt in lib.split("@")[1:]:  # lib.so@identity or lib.so@ENV=VAL
                k, _, v = opt.partition("=")
                env.update({k: v} if v else {"IVHD_ORDER": k})
            r = subprocess.run([sys.executable, __file__, "--child", "300", kind, str(m)], env=env,
                               capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-800:], flush=True)

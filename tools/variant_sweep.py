"""Time the step kernel of several library builds (tools/build_variant.py)
on the C3 fixture and a planted 10^7 graph: us per iteration, steady state.

    python tools/variant_sweep.py sweep/lib_a.so sweep/lib_b.so ...
(each build runs in its own process; the product library is the default)."""
import json, os, subprocess, sys, time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C3 = os.path.join(ROOT, "tests", "golden", "c3_graph.npz")
CHILD = r'''
import os, sys, time, json
import numpy as np
sys.path.insert(0, ROOT)
import paper_2303_05455_b200._lib as L
L.LIB_PATH = LIB
import torch
from paper_2303_05455_b200 import synth
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
out = {}
for name in GRAPHS:
    if name == "c3":
        nb = np.load(C3)["neighbors"]
    elif name.startswith("npz:"):
        nb = np.load(os.path.join(os.path.dirname(C3), name[4:]))["neighbors"][:, :2]
    else:  # planted:M (nn=2) or plantedK:M (nn=K)
        kind, mm = name.split(":")
        nb = synth.planted_graph(int(mm), int(kind[7:] or 2), seed=0)
    m = nb.shape[0]
    rng = np.random.default_rng(0)
    y0 = init_layout(m, 2, rng); rn = sample_random_neighbors(m, nb, RN, rng)
    dev = DeviceEmbedding(m, 2)
    if MODE == "peer1":  # the fused peer exchange with one rank (sharded kernels + finalizer)
        tv, nt = dev.tiles()
        dev.shard_set_range(0, tv * nt)
        dev.peer_import([dev.peer_export(1, 0)])
    dev.set_optimizer(resolve_optimizer("force-directed", m)); dev.set_positions(y0); dev.set_graph(0, nb, rn)
    if MODE in ("auto", "grid") and hasattr(dev, "set_launch_mode"):
        dev.set_launch_mode(MODE)
    if L2G:  # driver-level L2 fetch granularity limit (CU_LIMIT_MAX_L2_FETCH_GRANULARITY)
        import ctypes
        cu = ctypes.CDLL("libcuda.so.1"); val = ctypes.c_size_t(0)
        cu.cuCtxGetLimit(ctypes.byref(val), 5); before = val.value
        rc = cu.cuCtxSetLimit(5, ctypes.c_size_t(L2G)); cu.cuCtxGetLimit(ctypes.byref(val), 5)
        out[name + ":l2g"] = [before, rc, val.value]
    dev.snapshot()
    best = []
    for rep in range(4):
        dev.restore(); torch.cuda.synchronize(); t0 = time.perf_counter()
        dev.run(0, "l2", 0.1, ITERS); torch.cuda.synchronize()
        best.append((time.perf_counter() - t0) / ITERS * 1e6)
    out[name] = round(min(best[1:]), 2)
    if FLOOR:  # the gather-only pass over the same connections (ivhd_gather_floor)
        out[name + ":floor"] = round(dev.gather_floor(0), 2)
    dev.close()
print(json.dumps(out))
'''


def main():
    libs = sys.argv[1:] or [os.path.join(ROOT, "paper_2303_05455_b200", "libivhd_b200.so")]
    graphs = os.environ.get("GRAPHS", "c3,planted:10000000").split(",")
    iters = int(os.environ.get("ITERS", "500"))
    for lib in libs:
        root = ROOT
        if lib.endswith("/"):  # a package tree (another revision): its own python + library
            root = os.path.abspath(lib)
            lib = os.path.join(root, "paper_2303_05455_b200", "libivhd_b200.so")
        code = f"FLOOR={int(os.environ.get('FLOOR', '0'))}\nRN={int(os.environ.get('RN', '1'))}\nL2G={int(os.environ.get('L2G', '0'))}\nMODE={os.environ.get('MODE', '')!r}\nC3={C3!r}\nROOT={root!r}\nLIB={os.path.abspath(lib)!r}\nGRAPHS={graphs!r}\nITERS={iters}\n" + CHILD
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        print(os.path.basename(lib), r.stdout.strip() or r.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()

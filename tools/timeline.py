"""(PEER=1: the one-rank peer-exchange instantiation.)
Block timeline of two consecutive step-kernel launches (iterations 10, 11)
at C3, from a debug build:  python tools/build_variant.py tl -DIVHD_TIMELINE
then on the GPU box:  IVHD_B200_LIB=sweep/lib_tl.so python tools/timeline.py"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import synth
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding

kind = sys.argv[1] if len(sys.argv) > 1 else "mixture"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_400_000
cache = "/tmp/ivhd_c3_graph.npy"
if kind == "mixture":
    if not os.path.exists(cache):
        np.save(cache, synth.mixture_knn_graph(1_400_000, 100, k=2, seed=0)[0])
    nb = np.load(cache)
elif kind.endswith(".npz"):
    nb = np.load(kind)["neighbors"]
else:
    nb = synth.planted_graph(m, 2, seed=0)
m = nb.shape[0]
g = np.random.default_rng(0)
dev = DeviceEmbedding(m, 2)
if os.environ.get("PEER"):  # sharded kernels with the fused peer exchange, one rank
    tv, nt = dev.tiles()
    dev.shard_set_range(0, tv * nt)
    dev.peer_import([dev.peer_export(1, 0)])
dev.set_optimizer(resolve_optimizer("force-directed", m))
dev.init_positions(g)
dev.set_graph_sampled(0, nb[:, :2], 1, g)
dev.run(0, "l2", 0.1, 20)
lib = ctypes.CDLL(os.environ.get("IVHD_B200_LIB", os.path.join(os.path.dirname(__file__), "..", "paper_2303_05455_b200", "libivhd_b200.so")))
buf = np.zeros(2 * 1024 * 40, np.int64)
lib.ivhd_timeline_dump(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
t = buf.reshape(2, 1024, 40).astype(np.float64)
for it in range(2):
    T = t[it]
    live = T[:, 0] > 0
    T = T[live]
    base = T[:, 0].min()
    entry, dep, end = T[:, 0] - base, T[:, 1] - base, T[:, 38] - base
    units = T[:, 2:36]
    nu = (units > 0).sum(axis=1)
    prev = np.concatenate([T[:, 1:2], units], axis=1)
    dur = np.diff(prev, axis=1)[:, :34]
    dur = dur[(units > 0)]
    fin = T[:, 39].max() - base if (T[:, 39] > 0).any() else float("nan")
    print(f"iteration {10 + it}: blocks {live.sum()}  units/block {nu.min()}-{nu.max()} (mean {nu.mean():.1f})")
    print(f"  entry skew (ns): median {np.median(entry):.0f} max {entry.max():.0f}")
    print(f"  dependency wait done (ns): min {dep.min():.0f} median {np.median(dep):.0f} max {dep.max():.0f}")
    print(f"  first unit done (ns): median {np.median(units[:, 0] - base):.0f}")
    print(f"  unit duration (ns, warp 0): p10 {np.percentile(dur, 10):.0f} median {np.median(dur):.0f} p90 {np.percentile(dur, 90):.0f}")
    print(f"  loop end (ns): min {end.min():.0f} median {np.median(end):.0f} p90 {np.percentile(end, 90):.0f} max {end.max():.0f}")
    alld, arr = T[:, 36] - base, T[:, 37] - base
    print(f"  all warps done (ns): median {np.median(alld):.0f} max {alld.max():.0f};  arrival: max {arr.max():.0f}")
    print(f"  finalize end (ns): {fin:.0f}  (last arrival -> finalize end {fin - arr.max():.0f})")
    if it == 0:
        end0 = fin + base
nxt = t[1][t[1][:, 0] > 0]
print(f"gap: finalize end (it 10) -> first entry of it 11: {nxt[:, 0].min() - end0:.0f} ns; "
      f"-> median dependency release {np.median(nxt[:, 1]) - end0:.0f} ns")

"""Benchmark: IVHD edge-updates/s and seconds per 1.4M-vertex embed on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c3|c1|c2-adadelta|c2-nesterov|c4|c5]

Workload (BASELINE.json configs[2], "C3"): YAHOO-shaped synthetic kNN graph,
the exact 2-NN graph of M = 1.4M points of a 10-cluster Gaussian mixture in
100-D (spread 0.42, so the label metrics do not saturate: cf_10 = 0.76),
nn=2, rn=1, c=0.1, force-directed with the reference defaults, 2500
iterations, seed 0.  The graph is a committed fixture
(tests/golden/c3_graph.npz, built by the package's exact GPU kNN builder;
kNN construction is excluded from timing, as in the paper, and timed
separately in the `knn` leg, which also checks it rebuilds the fixture).

One "step" = one full 2500-iteration embed.  `value` = edge-updates/s with
the graph, positions and state resident in HBM (device-timed with CUDA
events on the launching stream; L2 flushed by a 256 MB write between
steps).  `e2e` = the same metric through the public API
`run_embedding(graph, config)` (N GPUs: `run_embedding_distributed`) from
host arrays in pinned memory (RNG setup, CSR build, H2D, loop, D2H).
`roofline` = algorithmic HBM bytes per iteration (8L + 36M
for force-directed) / device time per iteration.  `cpu_baseline` = the
reference package itself (`baseline/_ref`, ivhd.engine.run_embedding, all
host threads) on a bounded sample of the same workload.  `quality` = the
label neighbour hit and rank-curve summary of the e2e embedding beside the
reference's own full-run values (tests/golden/quality_c3.npz).

`--impl reference` times the UNMODIFIED reference package installed in
baseline/_ref (`ivhd.engine.run_embedding`, threads = all host cores) on the
same graph and config, rank 0 only; it never imports this package.

N > 1: `python bench.py --gpus N` starts N ranks itself (one process per
GPU) when it is not already running under torchrun; the ranks exchange
positions and partials through the fused NVLink path (sharded.py, no NCCL),
the gloo process group is the control plane only.
"""

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(ROOT, "tests", "golden")

METRIC = "IVHD edge-updates/s (1.4M-vertex YAHOO-shaped embed, nn=2 rn=1, 2500 iterations)"
UNIT = "edge-updates/s"

WORKLOADS = {
    # graph: committed fixture (tests/golden/<file>, key "neighbors") or "planted"
    "c3": dict(m=1_400_000, n=100, nn=2, rn=1, c=0.1, optimizer="force-directed", iterations=2500,
               graph="c3_graph.npz", spread=0.42, golden="quality_c3.npz",
               desc="YAHOO-shaped: exact 2-NN graph of a 1.4M x 100 ten-cluster mixture (spread 0.42)"),
    "c1": dict(m=20_000, n=784, nn=2, rn=1, c=0.01, optimizer="force-directed", iterations=2000,
               graph="c1_golden.npz", spread=0.23, golden="c1_golden.npz",
               desc="exact 2-NN graph of a 20k x 784 ten-cluster mixture (spread 0.23)"),
    "c2-adadelta": dict(m=70_000, n=784, nn=5, rn=1, c=0.01, optimizer="adadelta", iterations=2500,
                        graph="c2_golden.npz", golden="c2_golden.npz",
                        desc="MNIST-shaped: exact 5-NN graph of the reference's mnist_like(70000, 784)"),
    "c2-nesterov": dict(m=70_000, n=784, nn=5, rn=1, c=0.01, optimizer="nesterov", iterations=2500,
                        graph="c2_golden.npz", golden="c2_golden.npz",
                        desc="MNIST-shaped: exact 5-NN graph of the reference's mnist_like(70000, 784)"),
    "c4": dict(m=10_000_000, n=0, nn=3, rn=1, c=0.1, optimizer="force-directed", iterations=200,
               graph="planted", desc="planted-cluster kNN-shaped graph M=10^7 (synth.planted_graph)"),
    # the paper's 10^8+ scale (BASELINE configs[4] names 8 GPUs)
    "c5": dict(m=100_000_000, n=0, nn=2, rn=1, c=0.1, optimizer="force-directed", iterations=100,
               graph="planted", desc="planted-cluster kNN-shaped graph M=10^8 (synth.planted_graph)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def _synth():
    """synth.py loaded standalone (numpy only): the reference arm uses the same
    input generators without importing this package."""
    spec = importlib.util.spec_from_file_location("ivhd_b200_synth",
                                                  os.path.join(ROOT, "paper_2303_05455_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def make_graph(w):
    """The workload's kNN graph (input synthesis only, never timed)."""
    t0 = time.perf_counter()
    if w["graph"] == "planted":
        nb = _synth().planted_graph(w["m"], w["nn"], seed=0)
    else:
        nb = np.ascontiguousarray(np.load(os.path.join(GOLDEN, w["graph"]))["neighbors"], dtype=np.int32)
    assert nb.shape[0] == w["m"], (nb.shape, w["m"])
    log(f"[bench] graph {w['graph']} M={w['m']} ready in {time.perf_counter() - t0:.1f}s")
    return nb


def workload_config(args, w, world):
    return {"workload": f"{args.workload}: {w['desc']}, nn={w['nn']} rn={w['rn']} c={w['c']} "
                        f"{w['optimizer']}, {w['iterations']} iterations per step",
            "m": w["m"], "connections": (w["nn"] + w["rn"]) * w["m"],
            "iterations_per_step": w["iterations"],
            "parallelism": f"vertex-range shards x{world} (one process per GPU)" if world > 1 else "single GPU",
            "l2": "flushed between steps (256 MB write)"}


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """NVML clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = self.index  # CUDA ordinal -> NVML index through CUDA_VISIBLE_DEVICES
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis:
                ids = [v.strip() for v in vis.split(",")]
                if idx < len(ids) and ids[idx].isdigit():
                    idx = int(ids[idx])
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nv = nv
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.nv = None
        return self

    def _poll(self):
        nv = self.nv
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((float(sm), float(mx), [bool(r & b) for b in bits]))
            except Exception:
                pass
            self.stop.wait(0.01)

    def __exit__(self, *exc):
        if self.nv is not None:
            self.stop.set()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2][i]})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(workload):
    """DRAM bytes per launch of the step kernel from the newest committed ncu
    capture of THIS workload (profiles/rNN_<workload>_step_ncu.json, written by
    tools/ncu_to_profile.py); None for workloads without one."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r[0-9][0-9]_{workload}_step_ncu.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        return {"bytes_per_launch": d["dram_bytes_per_launch"], "source": "profiles/" + os.path.basename(files[-1]),
                "capture": d.get("capture", "")}
    except Exception:
        return None


# ------------------------------------------------------- the reference (CPU)


def _import_reference():
    """The unmodified reference package from baseline/_ref (pip-installed from
    /root/reference); None when it is not there."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ivhd")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import ivhd
    import ivhd.engine
    import ivhd.knng

    assert os.path.realpath(ivhd.__file__).startswith(os.path.realpath(ref)), ivhd.__file__
    return ivhd


class ReferenceTimer:
    """Times `ivhd.engine.run_embedding(graph, config, threads=all cores)` of
    the reference on the workload's graph; one call = `n` loop iterations (a
    bounded sample of the embed; its setup, _Run + RNG draws, is inside)."""

    def __init__(self, nb, w):
        self.ivhd = _import_reference()
        self.w = w
        self.threads = os.cpu_count() or 1
        self.L = (w["nn"] + w["rn"]) * w["m"]
        if self.ivhd is not None:
            self.kind = "reference"
            self.graph = self.ivhd.knng.KnnGraph(neighbors=nb, distances=np.zeros(nb.shape),
                                                 metric="euclidean")
        else:  # the oracle restatement (test infrastructure) only if baseline/_ref is missing
            self.kind = "port"
            self.nb = nb

    def call(self, n, threads=None):
        w = self.w
        threads = threads or self.threads
        t0 = time.perf_counter()
        if self.kind == "reference":
            E = self.ivhd.engine
            cfg = E.EmbeddingConfig(nn=w["nn"], rn=w["rn"], c=w["c"], iterations=n, seed=0,
                                    optimizer=w["optimizer"])
            E.run_embedding(graph=self.graph, config=cfg, threads=threads)
        else:
            sys.path.insert(0, ROOT)
            from oracle.ivhd_oracle import OracleRun

            OracleRun(self.nb, nn=w["nn"], rn=w["rn"], c=w["c"], iterations=n, seed=0,
                      optimizer=w["optimizer"], threads=threads).run()
        return time.perf_counter() - t0

    def pick_n(self, budget_s):
        """Iterations per call so one call takes about budget_s (from a 2-iteration probe)."""
        t2 = self.call(2)
        t1 = self.call(1)
        per = max(t2 - t1, 1e-4)
        return int(max(1, min(self.w["iterations"], round((budget_s - t1 + per) / per))))

    def describe(self, n, value):
        what = ("ivhd.engine.run_embedding from baseline/_ref (the unmodified reference package)"
                if self.kind == "reference" else "oracle port of the reference loop (baseline/_ref missing)")
        return {"value": value, "unit": UNIT, "cores": self.threads, "kind": self.kind,
                "sample": f"run_embedding(iterations={n}) per call (setup included) of the "
                          f"{self.w['iterations']}-iteration embed at M={self.w['m']}: {what}, threads={self.threads}"}


def reference_arm(args, w):
    """--impl reference: the reference's CPU implementation on all host cores."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    nb = make_graph(w)
    rt = ReferenceTimer(nb, w)
    n = args.ref_iters or rt.pick_n(args.ref_budget)
    for _ in range(args.warmup):
        rt.call(n)
    times = [rt.call(n) for _ in range(args.steps)]
    tot = sum(times)
    value = rt.L * n * args.steps / tot
    world = args.gpus
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic (the b200 arm's graph fixture / generator, same seed)",
        "config": workload_config(args, w, world),
        "s_per_embed_extrapolated": tot / (args.steps * n) * w["iterations"],
        "cpu_baseline": rt.describe(n, value),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm


def algorithmic_bytes(m, n_entries, optimizer):
    """col ids 4 B/entry + row_ptr 4 B/vertex + Y read and
    write 8+8 B/vertex + S*16 B/vertex of optimizer state (S=1 FD)."""
    s = {"force-directed": 1, "momentum": 1, "nesterov": 1, "sgd": 0, "adam": 2, "adadelta": 2}[optimizer]
    return 4 * n_entries + 4 * (m + 1) + 16 * m + 16 * s * m


def knn_leg(w, local, peaks, nb):
    """Time the GPU kNN builder (excluded from the embed
    timing, as in the paper) on the workload's point set, and check that it
    rebuilds the committed graph fixture."""
    from paper_2303_05455_b200 import knng, synth

    if "spread" not in w:
        return None
    x, _ = synth.mixture_points(w["m"], w["n"], seed=0, spread=w["spread"])
    x = x.astype(np.float64)
    best, g = None, None
    for _ in range(2):  # the first build also grows the stream-ordered memory pool
        t0 = time.perf_counter()
        g = knng.build_exact_knn(x, w["nn"], device=local)
        wall = time.perf_counter() - t0
        if best is None or wall < best[0]:
            best = (wall, dict(knng.last_stats))
    wall, st = best
    kp = (w["n"] + 7) // 8 * 8
    flops = 2.0 * w["m"] * w["m"] * kp
    peak = float(peaks.get("bf16_tflops", 1685.7)) / 2.0
    ach = flops / st["tc_seconds"] / 1e12
    return {"workload": f"exact kNN graph, M={w['m']} N={w['n']} k={w['nn']} (euclidean, fp64 input)",
            "s_per_build": wall, "tc_pass_s": st["tc_seconds"], "rerank_s": st["rerank_seconds"],
            "exact_rescan_rows": st["exact_rows"],
            "rebuilds_fixture": bool(np.array_equal(g.neighbors[:, : nb.shape[1]], nb)),
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                         "note": "tf32 tcgen05 candidate pass: 2*M^2*Kpad flops / pass time; peak = "
                                 "MEASURED_PEAKS.json bf16_tflops / 2 (dense tf32 rate is half of bf16)"}}


def quality_leg(w, points, local):
    """Label neighbour hit (all points) and rank curves (the reference's
    subsample) of the e2e embedding, beside the reference's own values."""
    from paper_2303_05455_b200 import metrics, synth

    if "golden" not in w:
        return None
    g = np.load(os.path.join(GOLDEN, w["golden"]))
    m = w["m"]
    if "labels" in g:
        labels = g["labels"].astype(np.int64)
    else:
        labels = synth.mixture_labels(m, w["n"], seed=0, spread=w["spread"])
    metrics.neighbor_hit(points[:4096], labels[:4096], nn_max=100, device=local)  # warm-up
    t0 = time.perf_counter()
    cf_nn, cf = metrics.neighbor_hit(points, labels, nn_max=100, device=local)
    q = {"neighbor_hit_cf": cf, "cf_2": float(cf_nn[1]), "cf_10": float(cf_nn[9]),
         "seconds": time.perf_counter() - t0,
         "note": "metrics.neighbor_hit(nn_max=100) of the e2e embedding on the GPU (exact grid kNN)"}
    pre = w["optimizer"] + "_" if w["optimizer"] + "_cf" in g else ""
    q["reference"] = {"neighbor_hit_cf": float(g[pre + "cf"]), "cf_2": float(g[pre + "cf_nn"][1]),
                      "cf_10": float(g[pre + "cf_nn"][9]), "stress": float(g[pre + "stress"]),
                      "source": f"tests/golden/{w['golden']} (reference ivhd.engine.run_embedding, fp64 CPU)"}
    if "summary_keys" in g and "spread" in w:
        sub = g["sub"] if "sub" in g else np.arange(m)
        x, _ = synth.mixture_points(m, w["n"], seed=0, spread=w["spread"])
        xs = x[sub].astype(np.float64)
        del x
        t0 = time.perf_counter()
        cur = metrics.evaluate_embedding(xs, points[sub], labels=labels[sub], nn_max=100, report_ks=(15, 100),
                                         device=local)
        q["curves"] = {**cur.summary(), "seconds": time.perf_counter() - t0,
                       "sample": f"{len(sub)} rows (the reference golden's subsample)",
                       "note": "metrics.evaluate_embedding on the GPU (curve pass k_max=1000)"}
        q["reference"]["curves"] = {str(k): float(v) for k, v in zip(g["summary_keys"], g["summary_vals"])}
    return q


def gpu_arm(args, w):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding
    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or args.sharded, f"WORLD_SIZE={world} but --gpus {args.gpus}"
    torch.cuda.set_device(local)
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if "MASTER_PORT" not in os.environ:
            import socket

            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(so.getsockname()[1])
        # control plane only (IPC handles, barriers, max over ranks): the fused
        # exchange moves the data itself, so the process group is gloo on the host
        dist.init_process_group("gloo")
    nb = make_graph(w)
    m, L, iters = w["m"], (w["nn"] + w["rn"]) * w["m"], w["iterations"]

    # same setup draws as run_embedding (engine.py:165, 214-215)
    rng = np.random.default_rng(0)
    nn_sets = nb[:, : w["nn"]]
    y0 = init_layout(m, 2, rng)
    rn = sample_random_neighbors(m, nn_sets, w["rn"], rng)

    stream = torch.cuda.Stream(device=local)  # the library launches on this stream
    torch.cuda.set_stream(stream)
    if sharded:
        from paper_2303_05455_b200.sharded import ShardedEmbedding

        dev = ShardedEmbedding(m, 2, rank, world, device=local, stream=stream.cuda_stream)
    else:
        dev = DeviceEmbedding(m, 2, device=local, stream=stream.cuda_stream)
    dev.set_optimizer(resolve_optimizer(w["optimizer"], m))
    dev.set_positions(y0)
    dev.set_graph(0, nn_sets, rn)
    dev.snapshot()
    n_entries = 2 * L
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def one_step():
        dev.restore()
        _, _, done, div = dev.run(0, "l2", w["c"], iters)
        assert done == iters and not div

    for _ in range(args.warmup):
        flush.zero_()
        one_step()
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between steps (outside the events)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            one_step()
            ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1) / 1e3)
    torch.cuda.synchronize()
    tot = sum(times)
    if sharded:
        t = torch.tensor([tot], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
        dist.barrier()
    value = L * iters * args.steps / tot
    s_iter = tot / (args.steps * iters)
    dev_launches = dev.launches_per_iteration() if hasattr(dev, "launches_per_iteration") else 1
    gfloor = None
    if not sharded:
        # the same neighbour gathers with nothing else (ivhd_gather_floor): the
        # memory-system floor of an iteration on this graph, beside the HBM roofline
        g_us = dev.gather_floor(0)
        gfloor = {"us_per_pass": g_us, "us_per_iteration": s_iter * 1e6, "frac": g_us / (s_iter * 1e6),
                  "entries_per_pass": n_entries,
                  "note": "one pass streaming the column ids and gathering every neighbour position "
                          "(no arithmetic, update or decision), CUDA events, warm L2, best of 10 in each of three sweeps (per-block slices at 8 and 3 blocks per SM, whole grid front to back); "
                          "frac = that floor / the step kernel's time per iteration"}
    nvlink = None
    if sharded and getattr(dev, "exchange", None) == "p2p":
        # fused exchange: position records this rank stores into peers per
        # iteration (halo masks) -> NVLink bytes; max over ranks
        recs, nbytes_pe = dev.device_embedding.peer_halo()
        t = torch.tensor([float(nbytes_pe), float(recs)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        allgather_bytes = (world - 1) * (m // world) * 8
        nvlink = {"exchange": "fused P2P stores from the step kernel (halo masks), no NCCL",
                  "bytes_per_iteration_per_rank_max": float(t[0]), "records_per_iteration_per_rank_max": float(t[1]),
                  "allgather_bytes_per_rank": allgather_bytes,
                  "achieved_gbs": float(t[0]) / s_iter / 1e9,
                  "peak_gbs": 770.0,
                  "note": "bytes each rank writes over NVLink per iteration / device time per iteration; "
                          "peak = measured peer copy per direction (B200_PROFILING.md)"}
    dev.close() if hasattr(dev, "close") else None

    # ---------------- e2e: public API from pinned host arrays
    e2e = None
    final_points = None
    final_stress = None
    if not args.no_e2e:
        nb_pinned = torch.empty(nb.shape, dtype=torch.int32, pin_memory=True).numpy()
        nb_pinned[...] = nb
        graph = KnnGraph(nb_pinned)
        cfg = EmbeddingConfig(nn=w["nn"], rn=w["rn"], c=w["c"], iterations=iters, seed=0,
                              optimizer=w["optimizer"])
        if sharded:
            from paper_2303_05455_b200.sharded import run_embedding_distributed

            call = lambda: run_embedding_distributed(graph=graph, config=cfg, device=local)  # noqa: E731
        else:
            call = lambda: run_embedding(graph=graph, config=cfg, device=local)  # noqa: E731
        walls = []
        for i in range(2 + args.e2e_steps):
            torch.cuda.synchronize()
            if sharded:
                dist.barrier()
            t0 = time.perf_counter()
            res = call()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            if sharded:
                t = torch.tensor([wall], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                wall = float(t.item())
            if i >= 2:  # two warm-up calls (allocator pools, pinned result buffers)
                walls.append(wall)
        final_stress = res.state.stress
        final_points = res.embedding.points
        # H2D: the nn-id block (the layout and random partners are drawn on the
        # device); D2H: positions (state + embedding) and deltas, the partners, the trace
        h2d = m * nb.shape[1] * 4
        d2h = 3 * m * 2 * 8 + m * w["rn"] * 4 + iters * 16
        e2e = {"value": L * iters / statistics.mean(walls), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "s_per_embed": statistics.mean(walls), "steps": len(walls)}

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        rt = ReferenceTimer(nb, w)
        n = rt.pick_n(args.cpu_budget / 3)
        ts = [rt.call(n) for _ in range(2)]
        cpu = rt.describe(n, rt.L * n * len(ts) / sum(ts))
        n1 = max(1, n // 4)  # the same on one thread (T=1 and T=all cores)
        cpu["value_1_thread"] = rt.L * n1 / rt.call(n1, threads=1)
        cpu["sample_1_thread"] = f"run_embedding(iterations={n1}), threads=1"
    knn = None
    if world == 1 and rank == 0 and not args.no_knn:
        knn = knn_leg(w, local, peaks, nb)
    quality = None
    if final_points is not None and rank == 0 and not args.no_quality:
        quality = quality_leg(w, final_points, local)

    if rank == 0:
        peak = float(peaks.get("hbm_gbs", 6550.0))
        nbytes = algorithmic_bytes(m, n_entries, w["optimizer"])
        achieved = nbytes / s_iter / 1e9
        tr = ncu_traffic(args.workload) or {}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong",  # one graph split over the ranks: total work fixed
            "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic: {w['desc']} (committed fixture / seeded generator; kNN untimed, "
                    "timed separately under 'knn')",
            "config": workload_config(args, w, world),
            "s_per_embed": tot / args.steps, "it_per_s": 1.0 / s_iter,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": tr.get("bytes_per_launch"),
                         "traffic_source": tr.get("source"), "traffic_capture": tr.get("capture"),
                         "algorithmic_bytes_per_launch": nbytes,
                         "note": f"algorithmic bytes {nbytes} per iteration (8L+36M for FD) / device time "
                                 "per iteration incl. inter-launch gaps; peak = MEASURED_PEAKS.json hbm_gbs"},
            "gather_floor": gfloor,
            "cpu_baseline": cpu, "e2e": e2e,
            # per step: one step-kernel launch per iteration, plus (one GPU) the
            # launch that decides the run's last iteration (deferred decisions)
            "gpu_launches": args.steps * (iters * dev_launches + (0 if sharded else 1)),
            "clocks": clk.summary(), "nvlink": nvlink,
            "final_stress_e2e": final_stress,
            "knn": knn, "quality": quality,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


def _spawned(rank, world, port, argv):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.argv = [sys.argv[0]] + argv
    main()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--iterations", type=int, default=None, help="override (profiling)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded) loop even on one GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-knn", action="store_true", help="skip the kNN-builder leg")
    ap.add_argument("--no-quality", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-iters", type=int, default=0, help="reference arm: iterations per step (0 = auto)")
    ap.add_argument("--ref-budget", type=float, default=3.0, help="reference arm: seconds per step (auto)")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.workload])
    if args.iterations:
        w["iterations"] = args.iterations
    if args.impl == "reference":
        return reference_arm(args, w)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not under torchrun: start one process per GPU ourselves
        import socket

        import torch.multiprocessing as mp

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        mp.start_processes(_spawned, args=(args.gpus, port, sys.argv[1:]), nprocs=args.gpus,
                           start_method="spawn", join=True)
        return 0
    return gpu_arm(args, w)


if __name__ == "__main__":
    sys.exit(main())

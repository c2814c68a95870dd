"""Vertex-range sharding of the IVHD loop across GPUs.

The update is synchronous (Jacobi): every force of iteration n is computed
from the same positions Y_n (engine.py:360-372), so vertex ranges are
independent given Y_n and one exchange per iteration suffices.

Each rank holds the full (relabelled) symmetrised CSR and a full replica of
the positions and updates the vertices of its tile-aligned range [v0, v1)
(equal tile counts; the vertex order deals the degree-sorted vertices over
8 rank groups so every range has the same edge count).  Two exchanges:

* "p2p" (default on GPUs) — the fused exchange of ivhd_peer_* (one process
  per GPU, one node): the step kernel stores each updated position straight
  into the replica of every peer whose rows gather it (halo masks) over
  NVLink (CUDA IPC mappings) as it is computed, so the transfer overlaps the
  update tile by tile; its last block stores the rank's partial into every
  peer, raises an arrival flag on every rank, waits for all ranks' flags and
  reduces the rank partials in rank order to the same decision everywhere.
  No NCCL, no host work per iteration: one launch per iteration, replayed
  from CUDA graphs.  Ranks that cannot map each other's memory fall back to
  "nccl".
* "nccl" — the step writes its slice locally, then the slice and the
  rank's tile partials are all-gathered in place through torch.distributed
  (NCCL; gloo in the CPU tests) and ivhd_shard_finalize reduces them.  Kept
  as the portable baseline and for the CPU tests.

Either way every rank reduces the same per-tile partials in the same order,
so the auto-adapt decision, the trace and the positions are identical on
all ranks and for every rank count.  The fused single-GPU loop sums
per-thread running partials instead, so its trace agrees with the sharded
one to fp32 summation order.
"""

import numpy as np

from .errors import InvalidArgumentError


def shard_ranges(n_tiles_cap, tile_v, world):
    """Equal tile counts per rank (the padded tile count is a multiple of 8)."""
    if world < 1 or n_tiles_cap % world:
        raise InvalidArgumentError(f"world size {world} must divide the padded tile count {n_tiles_cap}")
    per = n_tiles_cap // world
    return [(r * per * tile_v, (r + 1) * per * tile_v) for r in range(world)]


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class DeviceShardBackend:
    """The real backend: one DeviceEmbedding (C ABI) per rank."""

    def __init__(self, dev, stream=0):
        self.dev = dev
        self.stream = int(stream)

    def __getattr__(self, name):
        return getattr(self.dev, name)

    def _views(self, yptr=None):
        import torch

        if not hasattr(self, "_layout"):
            b = self.dev.shard_buffers()
            tile_v, n_tiles = self.dev.tiles()
            self._layout = (b, n_tiles * tile_v * b["floats_per_vertex"], n_tiles)
        b, n_floats, n_tiles = self._layout
        if yptr is None:  # synchronous path: the buffer the step wrote
            cur = self.dev.shard_buffers()["cur"]
            yptr = b["ybuf"][1 - cur]
        dev = torch.device("cuda", torch.cuda.current_device())
        ynext = torch.as_tensor(_CudaArray(yptr, n_floats, "<f4"), device=dev)
        parts = torch.as_tensor(_CudaArray(b["partials"], n_tiles * 4, "<f8"), device=dev)
        return ynext, parts

    def exchange_views(self, yptr=None):
        return self._views(yptr)


def _allgather_inplace(buf, rank, world, group=None):
    """All ranks contribute chunk `rank` of `buf`; afterwards every rank holds all chunks."""
    import torch
    import torch.distributed as dist

    chunk = buf.numel() // world
    mine = buf[rank * chunk:(rank + 1) * chunk]
    if buf.is_cuda:
        # NCCL runs in place when sendbuff == recvbuff + rank * count: no copy
        dist.all_gather_into_tensor(buf, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine.clone(), group=group)
        buf.copy_(torch.cat(parts))


def _peer_capable(device, group=None):
    """True on every rank iff all ranks share one host and every pair of
    their GPUs can access each other's memory (collective over `group`)."""
    import socket

    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    me = (socket.gethostname(), int(device))
    ranks = [None] * world
    dist.all_gather_object(ranks, me, group=group)
    ok = all(h == me[0] for h, _ in ranks) and all(
        d == me[1] or torch.cuda.can_device_access_peer(me[1], d) for _, d in ranks)
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok), group=group)
    return all(oks)


class ShardedEmbedding:
    """One rank's share of a distributed IVHD run (same surface as
    DeviceEmbedding for set-up; `run` drives the per-iteration exchange)."""

    def __init__(self, m, dim, rank, world, device=0, stream=0, group=None, backend=None, exchange=None):
        if backend is None:
            from .device import DeviceEmbedding

            backend = DeviceShardBackend(DeviceEmbedding(m, dim, device=device, stream=stream), stream)
            exchange = exchange or "p2p"
        self.exchange = exchange or "nccl"
        if self.exchange not in ("p2p", "nccl"):
            raise InvalidArgumentError(f"unknown exchange {exchange!r}")
        self.backend = backend
        self._graphs = {}
        self.m, self.dim, self.rank, self.world, self.group = int(m), int(dim), int(rank), int(world), group
        tile_v, n_tiles_cap = backend.tiles()
        self.ranges = shard_ranges(n_tiles_cap, tile_v, self.world)
        self.v0, self.v1 = self.ranges[self.rank]
        backend.shard_set_range(self.v0, self.v1)
        if self.exchange == "p2p" and self.world > 1 and not _peer_capable(device, group):
            # some pair of ranks cannot map each other's memory (another node,
            # no P2P path): every rank falls back to the NCCL all-gather
            import torch.distributed as dist

            self.exchange = "nccl"
            if dist.get_backend(group) != "nccl":
                self.group = group = dist.new_group(backend="nccl")
        if self.exchange == "p2p":
            # fused NVLink exchange (include/ivhd_b200.h ivhd_peer_*): every
            # rank publishes its buffers' CUDA IPC handles, opens the others'
            mine = backend.peer_export(self.world, self.rank)
            handles = [mine]
            if self.world > 1:
                import torch.distributed as dist

                handles = [None] * self.world
                dist.all_gather_object(handles, mine, group=group)
            backend.peer_import(handles)

    # set-up (graph, draws, optimizer, positions, read-back) is identical on
    # every rank: delegated to the rank's DeviceEmbedding
    def __getattr__(self, name):
        if name == "backend":
            raise AttributeError(name)
        return getattr(self.backend, name)

    @property
    def device_embedding(self):
        """The rank's DeviceEmbedding (None for a custom backend)."""
        return getattr(self.backend, "dev", None)

    def launches_per_iteration(self):
        """Kernels per iteration: p2p = the step kernel alone (it publishes to
        the peers, waits for their flags and decides in its last block; the
        finalizer kernel only exists for in-process emulated ranks); nccl =
        local update, tile fold, finalizer (NCCL's all-gathers come on top)."""
        return 1 if self.exchange == "p2p" else 3

    def step(self, slot, norm, c):
        """One synchronous iteration: local update, exchange, fixed-order
        decision read back to the host -> (stress, b, committed, diverged)."""
        self.backend.step_local(slot, norm, c)
        ynext, parts = self.backend.exchange_views()
        _allgather_inplace(ynext, self.rank, self.world, self.group)
        _allgather_inplace(parts, self.rank, self.world, self.group)
        return self.backend.step_finalize()

    def _iteration(self, slot, norm):
        be = self.backend
        yptr = be.shard_step(slot, norm)
        ynext, parts = be.exchange_views(yptr)
        _allgather_inplace(ynext, self.rank, self.world, self.group)
        _allgather_inplace(parts, self.rank, self.world, self.group)
        be.shard_finalize()

    def run(self, slot, norm, c, n_iter, graph_chunk=None):
        """Same contract as DeviceEmbedding.run: (stress[], step[], done, diverged).

        Asynchronous: per iteration the local update, the two all-gathers and
        the finalizer are queued on the stream without reading anything back
        (the exchange buffer alternates by parity, see ivhd_shard_step); the
        trace and the divergence status are read once at the end.  On CUDA the
        sequence of `graph_chunk` (even) iterations is captured once as a CUDA
        graph (kernels + NCCL collectives) and replayed, so the host issues one
        launch per chunk instead of ~5 calls per iteration."""
        be = self.backend
        if self.exchange == "p2p":  # the device drives the whole exchange
            return be.run(slot, norm, c, n_iter)
        n_iter = int(n_iter)
        parity, epoch = be.shard_begin(slot, c, n_iter)
        chunk = self.graph_chunk if graph_chunk is None else int(graph_chunk)
        chunk -= chunk % 2  # a replay must leave the buffer parity unchanged
        done = 0
        if chunk >= 2 and n_iter >= 3 + chunk and self._can_capture():
            key = (slot, norm, chunk)
            g = self._graphs.get(key)
            if g is not None and g[2] != epoch:  # CSR / optimizer / trace buffer changed
                g = None
            # warm-up (kernel attributes, NCCL communicator, allocator pools) and
            # alignment to the parity the cached graph was captured at
            warm = 2 if g is None else (0 if g[1] == parity else 1)
            for _ in range(warm):
                self._iteration(slot, norm)
            parity ^= warm & 1
            done = warm
            if g is None:
                g = (self._capture(chunk, slot, norm), parity, epoch)
                self._graphs[key] = g
            while n_iter - done >= chunk:
                g[0].replay()
                done += chunk
        for _ in range(n_iter - done):
            self._iteration(slot, norm)
        return be.shard_end()

    graph_chunk = 32

    def _can_capture(self):
        # the context must launch on the caller's stream (not a private one)
        try:
            import torch

            return (isinstance(self.backend, DeviceShardBackend) and self.backend.stream != 0
                    and torch.cuda.is_available())
        except Exception:
            return False

    def _capture(self, chunk, slot, norm):
        import torch

        stream = torch.cuda.ExternalStream(self.backend.stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(chunk):
                    self._iteration(slot, norm)
        return g


def run_embedding_distributed(graph=None, config=None, dataset=None, helper_graph=None, group=None,
                              device=None):
    """`run_embedding` (engine.py:312-414) across the ranks of a
    torch.distributed process group, one GPU per rank: every rank calls it
    with the same graph and config and gets the same RunResult (the full
    embedding is replicated on every rank).  Observers are not supported
    here (the steering server drives one GPU)."""
    import torch
    import torch.distributed as dist

    from .config import coerce_config
    from .embed import _drive, _Session

    config = coerce_config(config)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        device = torch.cuda.current_device()
    stream = torch.cuda.current_stream(device)
    if stream.cuda_stream == 0:  # graph capture needs a real stream
        stream = torch.cuda.Stream(device=device)

    def make(m, dim, device=device):
        return ShardedEmbedding(m, dim, rank, world, device=device, stream=stream.cuda_stream, group=group)

    with torch.cuda.stream(stream):
        sess = _Session(graph, config, dataset, helper_graph, device, make_device=make)
        if world > 1:  # every rank draws the directions of all ranks' degenerate pairs, in one order
            def gathered(slot, rows, entries):
                parts = [None] * world
                dist.all_gather_object(parts, (np.asarray(rows).tolist(), np.asarray(entries).tolist()), group=group)
                return sess.degenerate_directions(slot, sum((p[0] for p in parts), []),
                                                  sum((p[1] for p in parts), []))

            sess.dev.device_embedding.degenerate_resolver = gathered
        return _drive(sess, config, None)

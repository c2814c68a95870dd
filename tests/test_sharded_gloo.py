"""The multi-GPU driver (paper_2303_05455_b200/sharded.py) on CPU: two gloo
ranks exchange position slices and tile partials exactly as the NCCL path
does.  The per-rank compute is a numpy stand-in backend built from the CPU
oracle (test infrastructure) with the library's tile/partial/decision
contract, so the test checks the sharding, exchange and fixed-order decision
logic: every rank ends bit-identical, a 2-rank run is bit-identical to a
1-rank run, and both follow the oracle's force-directed trajectory."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from oracle.ivhd_oracle import OracleRun
from paper_2303_05455_b200.sharded import ShardedEmbedding

TILE = 256


class NumpyShardBackend:
    """CPU stand-in for DeviceShardBackend (float64, force-directed)."""

    def __init__(self, m, conn, a=0.99, b=0.002, tau=None, c=0.1):
        self.m, self.conn, self.c = m, conn, c
        self.a, self.b, self.tau = a, b, 1e-3 * m if tau is None else tau
        self.n_tiles_cap = ((m + TILE - 1) // TILE + 7) // 8 * 8
        cap = self.n_tiles_cap * TILE
        self.Y = [torch.zeros(cap * 2, dtype=torch.float64), torch.zeros(cap * 2, dtype=torch.float64)]
        self.delta = np.zeros((cap, 2))
        self.parts = torch.zeros(self.n_tiles_cap * 4, dtype=torch.float64)
        self.cur = 0
        self.csr = O.symmetrise(conn, m)

    def tiles(self):
        return TILE, self.n_tiles_cap

    def shard_set_range(self, v0, v1):
        self.v0, self.v1 = v0, v1

    def set_positions(self, y):
        self.Y[self.cur][: self.m * 2] = torch.from_numpy(np.asarray(y, dtype=np.float64).ravel())

    def positions(self):
        return self.Y[self.cur][: self.m * 2].numpy().reshape(self.m, 2).copy()

    def step_local(self, slot, norm, c):
        y = self.positions()
        f, _ = O.csr_forces(y, self.csr, self.conn, self.c, norm)
        row_ptr, other, cidx = self.csr
        rows = np.repeat(np.arange(self.m), np.diff(row_ptr))
        d = np.sqrt(((y[rows] - y[other]) ** 2).sum(axis=1))
        w = self.conn.weights(self.c)[cidx]
        e_row = np.bincount(rows, weights=w * (self.conn.target[cidx] - d) ** 2, minlength=self.m)
        ynext = self.Y[1 - self.cur].numpy().reshape(-1, 2)
        parts = self.parts.numpy().reshape(-1, 4)
        for t in range(self.v0 // TILE, self.v1 // TILE):
            lo, hi = t * TILE, min((t + 1) * TILE, self.m)
            acc = np.zeros(4)
            for v in range(lo, hi):
                old = self.delta[v].copy()
                new = self.a * old + self.b * f[v]
                self.delta[v] = new
                ynext[v] = y[v] + new
                acc += [e_row[v], new @ new, old @ old, 0.0 if np.isfinite(ynext[v]).all() else 1.0]
            parts[t] = acc

    def exchange_views(self, token=None):
        return self.Y[1 - self.cur if token is None else token], self.parts

    # asynchronous contract (ivhd_shard_*): read Y[cur], write Y[cur^1], the
    # finalizer makes the written buffer current and refills it on rollback
    def shard_begin(self, slot, c, n_iter):
        self.trace, self.status, self.diverged_at = [], 0, None
        self.shard_cur = self.cur
        return self.cur, 0

    def shard_step(self, slot, norm):
        if not self.status:
            self.step_local(slot, norm, self.c)
        return self.shard_cur ^ 1

    def shard_finalize(self):
        out = self.shard_cur ^ 1
        self.shard_cur = out
        if self.status:
            return
        before = self.cur
        e, b, commit, div = self.step_finalize()
        self.trace.append((e, b))
        if div:
            self.status, self.diverged_at = 1, len(self.trace) - 1
            self.cur = before
            return
        if not commit:  # refill the written buffer with the unchanged positions
            self.Y[out][:] = self.Y[before]
        self.cur = out

    def shard_end(self):
        st = np.array([t[0] for t in self.trace])
        bb = np.array([t[1] for t in self.trace])
        if self.status:
            return st, bb, self.diverged_at, True
        return st, bb, len(self.trace), False

    def step_finalize(self):
        s = self.parts.numpy().reshape(-1, 4).sum(axis=0)
        E, dT = 0.5 * s[0], s[1] - s[2]
        commit = True
        if dT > self.tau:
            self.b *= 0.9
            commit = False
        elif dT < -self.tau:
            self.b *= 1.1
            commit = False
        if commit:
            self.cur ^= 1
        return E, self.b, commit, False


def _problem(m=700, seed=0, integ=None):
    rng = np.random.default_rng(seed)
    nb = ((np.arange(m)[:, None] + rng.integers(1, 30, size=(m, 2))) % m).astype(np.int32)
    orc = OracleRun(nb, nn=2, rn=1, c=0.1, iterations=30, seed=seed, integrator=integ)
    return nb, orc


def _worker(rank, world, port, iters, out, integ=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nb, orc = _problem(integ=integ)
        be = NumpyShardBackend(orc.m, orc.full, **(integ or {}))
        sh = ShardedEmbedding(orc.m, 2, rank, world, backend=be)
        sh.set_positions(orc.Y)
        stress, steps, done, div = sh.run(0, "l2", 0.1, iters)
        np.savez(os.path.join(out, f"rank{rank}_of{world}.npz"), y=sh.positions(), stress=stress, b=steps)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_two_gloo_ranks_match_one_rank_and_oracle(tmp_path):
    iters = 12
    for world in (1, 2):
        mp.start_processes(_worker, args=(world, _free_port(), iters, str(tmp_path)), nprocs=world,
                           start_method="spawn", join=True)
    r1 = np.load(tmp_path / "rank0_of1.npz")
    a = np.load(tmp_path / "rank0_of2.npz")
    b = np.load(tmp_path / "rank1_of2.npz")
    # every rank holds the same positions and the same trace ...
    np.testing.assert_array_equal(a["y"], b["y"])
    np.testing.assert_array_equal(a["stress"], b["stress"])
    np.testing.assert_array_equal(a["b"], b["b"])
    # ... bit-identical to the unsharded run (tile order is rank-independent)
    np.testing.assert_array_equal(a["y"], r1["y"])
    np.testing.assert_array_equal(a["stress"], r1["stress"])
    # ... and equal to the oracle's force-directed trajectory (float64)
    _, orc = _problem()
    for _ in range(iters):
        orc.step()
    np.testing.assert_allclose(a["y"], orc.Y, rtol=0, atol=1e-12)
    np.testing.assert_allclose(a["stress"], orc.trace_stress, rtol=1e-12)
    np.testing.assert_allclose(a["b"], orc.trace_b, rtol=1e-14)


@pytest.mark.timeout(300)
def test_async_loop_rollbacks_match_oracle(tmp_path):
    """Rollback-heavy auto-adapt (tiny tau, large b): the asynchronous loop's
    parity buffers and rollback refill follow the oracle on 1 and 2 ranks."""
    iters, integ = 12, {"b": 0.5, "tau": 1e-6}
    for world in (1, 2):
        mp.start_processes(_worker, args=(world, _free_port(), iters, str(tmp_path), integ), nprocs=world,
                           start_method="spawn", join=True)
    r1 = np.load(tmp_path / "rank0_of1.npz")
    a = np.load(tmp_path / "rank0_of2.npz")
    np.testing.assert_array_equal(a["y"], r1["y"])
    np.testing.assert_array_equal(a["b"], r1["b"])
    _, orc = _problem(integ=integ)
    for _ in range(iters):
        orc.step()
    b = np.asarray(orc.trace_b)
    assert (b[1:] != b[:-1]).sum() >= 3, "expected several auto-adapt rollbacks"
    np.testing.assert_allclose(a["y"], orc.Y, rtol=0, atol=1e-12)
    np.testing.assert_allclose(a["b"], b, rtol=1e-14)


def test_shard_plan_covers_all_vertices():
    be = NumpyShardBackend(700, _problem()[1].full)
    spans = [ShardedEmbedding(700, 2, r, 4, backend=NumpyShardBackend(700, be.conn)) for r in range(4)]
    covered = sorted((s.v0, s.v1) for s in spans)
    assert covered[0][0] == 0 and covered[-1][1] >= 700
    assert all(covered[i][1] == covered[i + 1][0] for i in range(3))


def _capable_worker(rank, world, port, out, deny_rank, host_of):
    """Runs sharded._peer_capable with a patched P2P query / host name."""
    import socket as _socket

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_05455_b200 import sharded

        torch.cuda.can_device_access_peer = lambda a, b: rank != deny_rank
        _socket.gethostname = lambda: host_of[rank]
        ok = sharded._peer_capable(device=rank)
        np.save(os.path.join(out, f"cap{rank}.npy"), np.array([ok]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("deny_rank,hosts,expect", [(-1, ("a", "a"), True), (1, ("a", "a"), False),
                                                    (-1, ("a", "b"), False)])
def test_peer_capability_is_agreed_by_every_rank(tmp_path, deny_rank, hosts, expect):
    """The fused exchange needs every pair of ranks to map each other's memory:
    one rank without a P2P path (or on another host) sends all ranks to the
    NCCL exchange, and every rank reaches the same answer."""
    mp.start_processes(_capable_worker, args=(2, _free_port(), str(tmp_path), deny_rank, hosts), nprocs=2,
                       start_method="spawn", join=True)
    got = [bool(np.load(tmp_path / f"cap{r}.npy")[0]) for r in range(2)]
    assert got == [expect, expect]

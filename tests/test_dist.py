"""CPU: the multi-GPU orchestration (paper_1505_04086_b200/dist.py) with
world size 2 over gloo.  The per-rank compute is a checker backend with the
same contract as DeviceOps (test infrastructure: plain sequential restatements
of K1-on-a-range, detect and detect-and-recolour), so what is tested here is
the distributed protocol: partitioning, slice all-gather, delta exchange,
global termination, and that every replica ends with the same proper
colouring within the degree bound."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1505_04086_b200 import dist as gdist


class CheckerOps:
    """Sequential CPU restatement of the per-rank ops (degree_id rule)."""

    def __init__(self, off: np.ndarray, cols: np.ndarray):
        self.off, self.cols = off, cols
        self.deg = np.diff(off)

    def _ff(self, colors, v, lower_only):
        nb = self.cols[self.off[v]:self.off[v + 1]]
        if lower_only:
            nb = nb[nb < v]
        used = set(int(c) for c in colors[nb].tolist() if 0 <= c <= self.deg[v])
        c = 0
        while c in used:
            c += 1
        return c

    def _defective(self, colors, v):
        cv = int(colors[v])
        if cv == -1:
            return False
        for w in self.cols[self.off[v]:self.off[v + 1]]:
            if int(colors[w]) == cv and (self.deg[v], v) < (self.deg[w], int(w)):
                return True
        return False

    def k1_range(self, colors, lo, hi):
        for v in range(lo, hi):
            colors[v] = self._ff(colors, v, True)
        return 0.0

    def detect_range(self, colors, lo, hi):
        return torch.tensor([v for v in range(lo, hi) if self._defective(colors, v)],
                            dtype=torch.int32)

    def round_list(self, colors, work):
        out = []
        for v in work.tolist():
            if self._defective(colors, v):
                colors[v] = self._ff(colors, v, False)
                out.append(v)
        return torch.tensor(out, dtype=torch.int32)

    def scatter(self, colors, ids, vals):
        colors[ids.long()] = vals


class CheckerPushOps(CheckerOps):
    """Push mode on CPU: every rank's replica is a shared-memory tensor and a
    commit writes all of them (the CPU stand-in for the peer stores)."""

    def __init__(self, off, cols, replicas, rank, world):
        super().__init__(off, cols)
        self.reps, self.rank, self.world = replicas, rank, world
        self.pairs = []

    def partition(self, rank, world, peer_ptrs):
        assert (rank, world) == (self.rank, self.world)

    def _commit(self, v, c):
        for r in self.reps:
            r[v] = c

    def k1_owned(self, colors):
        n = colors.numel()
        self.pairs = []
        for c0 in range(self.rank * gdist.CHUNK, n, self.world * gdist.CHUNK):
            for v in range(c0, min(c0 + gdist.CHUNK, n)):
                nb = self.cols[self.off[v]:self.off[v + 1]]
                nb = nb[nb < v]
                seen = colors[nb].tolist()
                self.pairs += [(int(u), v) for u, cu in zip(nb, seen) if cu == -1]
                used = set(c for c in seen if 0 <= c <= self.deg[v])
                c = 0
                while c in used:
                    c += 1
                self._commit(v, c)
        return 0.0

    def candidates(self, colors):
        out = set()
        for u, v in self.pairs:
            if int(colors[u]) == int(colors[v]):
                out.add(u if (self.deg[u], u) < (self.deg[v], v) else v)
        return torch.tensor(sorted(out), dtype=torch.int32)

    def round_list(self, colors, work):
        out = []
        for v in work.tolist():
            if self._defective(colors, v):
                self._commit(v, self._ff(colors, v, False))
                out.append(v)
        return torch.tensor(out, dtype=torch.int32)


def _graph(seed, n, avg):
    from paper_1505_04086_b200 import gcol
    rng = np.random.default_rng(seed)
    e = rng.integers(0, n, size=(int(n * avg / 2), 2))
    return gcol.build_graph(e, n)


def _worker(rank, world, port, seed, n, avg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(seed, n, avg)
        ops = CheckerOps(g.offsets(), g.adjacency())
        colors = torch.full((n,), -1, dtype=torch.int32)
        st = gdist.color_rsoc_distributed(ops, colors, n, rank, world)
        q.put((rank, colors.numpy().copy(), st.rounds, st.conflicts_per_round,
               st.round1_candidates))
    finally:
        dist.destroy_process_group()


def _push_worker(rank, world, port, seed, n, avg, reps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(seed, n, avg)
        ops = CheckerPushOps(g.offsets(), g.adjacency(), reps, rank, world)
        st = gdist.color_rsoc_partitioned(ops, reps[rank], n, rank, world, peer_ptrs=[0] * world)
        q.put((rank, reps[rank].numpy().copy(), st.rounds, st.conflicts_per_round,
               st.round1_candidates))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("seed,n,avg", [(1, 700, 6.0), (2, 1500, 12.0), (3, 257, 3.0)])
def test_partitioned_rsoc_world2(seed, n, avg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, n, avg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    (_, c0, r0, cpr0, cand0), (_, c1, r1, cpr1, cand1) = res
    assert np.array_equal(c0, c1), "replicas diverged"
    assert (r0, cpr0) == (r1, cpr1)
    g = _graph(seed, n, avg)
    off, cols = g.offsets(), g.adjacency()
    deg = np.diff(off)
    assert (c0 >= 0).all() and (c0 <= deg).all()
    rows = np.repeat(np.arange(n), deg)
    assert not (c0[rows] == c0[cols]).any(), "monochromatic edge"
    assert cpr0[-1] == 0 and r0 == len(cpr0)
    # the cross-rank boundary produced work for round 1 (the exchange matters)
    assert cand0 == cand1


def test_partition_bounds():
    for n in (0, 1, 255, 256, 257, 10_000, 1_000_003):
        for w in (1, 2, 3, 8):
            parts = gdist.partition(n, w)
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            assert all(lo % 256 == 0 for lo, _ in parts)


@pytest.mark.parametrize("seed,n,avg,world", [(4, 900, 6.0, 2), (5, 2000, 14.0, 2), (6, 1300, 5.0, 3),
                                               (7, 200, 5.0, 2)])
def test_push_mode_world(seed, n, avg, world):
    """Push mode: interleaved 256-id chunks, commits written into every
    replica, candidates gathered once, count all-reduced per round.  n = 200:
    one chunk, so nothing is read in flight and the empty-candidate exit
    (one all-reduce, rounds = 1) runs."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    reps = [torch.full((n,), -1, dtype=torch.int32).share_memory_() for _ in range(world)]
    procs = [ctx.Process(target=_push_worker, args=(r, world, port, seed, n, avg, reps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c0 = res[0][1]
    for r in res[1:]:
        assert np.array_equal(c0, r[1]), "replicas diverged"
        assert (r[2], r[3], r[4]) == (res[0][2], res[0][3], res[0][4])
    g = _graph(seed, n, avg)
    off, cols = g.offsets(), g.adjacency()
    deg = np.diff(off)
    assert (c0 >= 0).all() and (c0 <= deg).all()
    rows = np.repeat(np.arange(n), deg)
    assert not (c0[rows] == c0[cols]).any(), "monochromatic edge"
    assert res[0][3][-1] == 0 and res[0][2] == len(res[0][3])


def test_owner_of_interleaves_chunks():
    ids = torch.arange(0, 4096)
    own = gdist.owner_of(ids, 4)
    assert own[:256].eq(0).all() and own[256:512].eq(1).all() and own[1024:1280].eq(0).all()

"""Multi-GPU RSOC: 1-D vertex partition, replicated colours.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the
collectives).  Rank r owns the id range [lo_r, hi_r) -- contiguous ranges of
whole 256-id chunks, balanced by vertex count (ids are random, so edges
balance in expectation) -- and keeps a full replica of the colour array:

  1. K1 on the owned rows (gcol_cuda_k1_range), reading remote colours as
     they are in the replica (uncoloured at first);
  2. all-gather of the owned slices -> every replica complete;
  3. round 1: owned defective vertices (gcol_cuda_detect_range);
  4. each round: fused detect-and-recolour over the owned worklist
     (gcol_cuda_round_list), then an all-gather of the (id, colour) deltas
     (counts first, then padded lists) applied to every replica
     (gcol_cuda_scatter_colors); the global sum of recolours decides
     termination (conflicts_per_round is that sum, as in finish_round,
     parallel.hpp:140-154).

Correctness follows the single-GPU argument: inside a round
the remote part of a replica is stable, so a recolour avoids every stable
neighbour, and two vertices recoloured in the same round on different ranks
are both re-checked by their owners in the next round; the maximum-priority
vertex recoloured in a round never recolours again.

`ops` is the per-rank compute backend.  The product uses DeviceOps (the C
ABI on the rank's GPU); tests/test_dist.py runs the same orchestration on
CPU with a checker backend over gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

CHUNK = 256


def partition(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, chunk-aligned owned ranges [lo, hi) for every rank."""
    nch = (n + CHUNK - 1) // CHUNK
    bounds = [min(n, ((nch * r) // world) * CHUNK) for r in range(world + 1)]
    bounds[-1] = n
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


@dataclass
class DistStats:
    rounds: int = 0
    conflicts_per_round: List[int] = field(default_factory=list)
    conflicts_total: int = 0
    barrier_events: int = 0
    round1_candidates: int = 0
    k1_ms: float = 0.0
    exchanged_ids: int = 0


class DeviceOps:
    """Per-rank compute on the GPU through libgcol_cuda (device pointers)."""

    def __init__(self, graph, priority: int = 0, opt=None):
        from . import _lib, gcol
        self._lib = _lib
        self._gcol = gcol
        self.g = graph
        self.h = graph.handle()
        self.priority = int(priority)
        self.opt = opt or gcol.ParallelOptions()

    def _check(self, rc):
        self._gcol._check(rc)

    def k1_range(self, colors: torch.Tensor, lo: int, hi: int) -> float:
        st = self._lib.Stats()
        o = self.opt.to_c(1)
        self._check(self._lib.LIB.gcol_cuda_k1_range(self.h, C.byref(o), C.c_void_p(colors.data_ptr()),
                                                     lo, hi, C.byref(st)))
        return st.initial_pass_ns / 1e6

    def detect_range(self, colors: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
        out = torch.empty(max(hi - lo, 1), dtype=torch.int32, device=colors.device)
        n = C.c_int64(0)
        self._check(self._lib.LIB.gcol_cuda_detect_range(self.h, self.priority,
                                                         C.c_void_p(colors.data_ptr()), lo, hi,
                                                         C.c_void_p(out.data_ptr()), C.byref(n)))
        return out[:n.value]

    def round_list(self, colors: torch.Tensor, work: torch.Tensor) -> torch.Tensor:
        out = torch.empty(max(work.numel(), 1), dtype=torch.int32, device=colors.device)
        n = C.c_int64(0)
        if work.numel():
            self._check(self._lib.LIB.gcol_cuda_round_list(
                self.h, self.priority, C.c_void_p(colors.data_ptr()), C.c_void_p(work.data_ptr()),
                work.numel(), C.c_void_p(out.data_ptr()), C.byref(n)))
        return out[:n.value]

    def scatter(self, colors: torch.Tensor, ids: torch.Tensor, vals: torch.Tensor) -> None:
        if ids.numel():
            self._check(self._lib.LIB.gcol_cuda_scatter_colors(
                self.h, C.c_void_p(colors.data_ptr()), C.c_void_p(ids.data_ptr()),
                C.c_void_p(vals.data_ptr()), ids.numel()))


def _all_gather_var(t: torch.Tensor, world: int, group) -> List[torch.Tensor]:
    """All-gather of variable-length 1-D int32 tensors (counts, then padded)."""
    cnt = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    sizes = [int(c.item()) for c in counts]
    mx = max(sizes) if sizes else 0
    if mx == 0:
        return [t.new_empty(0) for _ in range(world)]
    pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
    pad[:t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:s] for o, s in zip(outs, sizes)]


def color_rsoc_distributed(ops, colors: torch.Tensor, n: int, rank: int, world: int,
                           group=None, round_cap: int = 1000) -> DistStats:
    """Partitioned RSOC; `colors` (int32[n], -1 filled) is this rank's
    replica and holds the full final colouring on return, on every rank."""
    st = DistStats()
    parts = partition(n, world)
    lo, hi = parts[rank]
    st.k1_ms = ops.k1_range(colors, lo, hi)
    # owned slices -> every replica (padded equal-size all-gather)
    span = max(h - l for l, h in parts) if parts else 0
    mine = torch.full((span,), -1, dtype=colors.dtype, device=colors.device)
    mine[:hi - lo] = colors[lo:hi]
    slices = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(slices, mine, group=group)
    for r, (l, h) in enumerate(parts):
        if r != rank and h > l:
            colors[l:h] = slices[r][:h - l]
    del slices, mine
    work = ops.detect_range(colors, lo, hi)
    cnt = torch.tensor([work.numel()], dtype=torch.int64, device=colors.device)
    dist.all_reduce(cnt, group=group)
    st.round1_candidates = int(cnt.item())
    while True:
        rec = ops.round_list(colors, work)
        vals = colors[rec.long()] if rec.numel() else rec
        ids_all = _all_gather_var(rec, world, group)
        vals_all = _all_gather_var(vals.to(torch.int32), world, group)
        found = sum(int(x.numel()) for x in ids_all)
        for r in range(world):
            if r != rank and ids_all[r].numel():
                ops.scatter(colors, ids_all[r], vals_all[r])
        st.exchanged_ids += found
        st.rounds += 1
        st.conflicts_per_round.append(found)
        st.conflicts_total += found
        if found == 0:
            break
        if st.rounds >= round_cap:
            raise RuntimeError("round_cap reached (no CPU repair fallback)")
        work = rec
    st.barrier_events = st.rounds + 1
    return st

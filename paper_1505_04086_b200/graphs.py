"""Seeded synthetic graphs for the five BASELINE.json configurations.

Stand-ins for the paper's datasets (UF meshes and R-MAT
ER/G/B, not in this container): same shapes, sizes and degree laws, with
vertex ids randomly permuted like the reference's shuffle_vertices
(rmat.hpp:144-155; "randomly shuffling vertex indices").

Every generator is counter-based (splitmix64 of the sample index), so the
output depends only on (parameters, seed) -- not on the device or on
thread counts -- and runs on CPU (tests) or CUDA (bench) through the same
torch code.  CSR construction is the canonical one of build_graph
(graph.hpp:98-138): loops dropped, duplicates collapsed, rows sorted.
This is workload generation, not the hot path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import torch

_M1 = 0xBF58476D1CE4E5B9 - (1 << 64)
_M2 = 0x94D049BB133111EB - (1 << 64)
_GOLD = 0x9E3779B97F4A7C15 - (1 << 64)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 (two's complement) by k."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def mix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    x = x ^ _srl(x, 30)
    x = x * _M1
    x = x ^ _srl(x, 27)
    x = x * _M2
    return x ^ _srl(x, 31)


def _stream(seed: int, idx: torch.Tensor, lane: int = 0) -> torch.Tensor:
    base = mix64(torch.tensor([seed * 0x100000001B3 + lane * 7919], dtype=torch.int64,
                              device=idx.device))
    return mix64(idx * _GOLD + base)


def uniform_below(seed: int, idx: torch.Tensor, bound: int, lane: int = 0) -> torch.Tensor:
    return _srl(_stream(seed, idx, lane), 11) % bound


def uniform01(seed: int, idx: torch.Tensor, lane: int = 0) -> torch.Tensor:
    return _srl(_stream(seed, idx, lane), 11).to(torch.float64) * (2.0 ** -53)


def random_permutation(n: int, seed: int, device) -> torch.Tensor:
    """perm[old] = new, a uniform permutation (sort of random keys)."""
    idx = torch.arange(n, dtype=torch.int64, device=device)
    keys = _srl(_stream(seed, idx, 99), 1)
    order = torch.argsort(keys)
    perm = torch.empty_like(order)
    perm[order] = idx
    return perm


def csr_from_edges(u: torch.Tensor, v: torch.Tensor, n: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """Canonical CSR (build_graph, graph.hpp:98-138) from undirected pairs:
    int64 offsets (n+1), int32 columns, rows sorted ascending."""
    device = u.device
    keep = u != v
    u, v = u[keep], v[keep]
    lo = torch.minimum(u, v)
    hi = torch.maximum(u, v)
    del u, v, keep
    key = torch.unique(lo * n + hi)  # sorted, deduplicated
    del lo, hi
    lo, hi = key // n, key % n
    del key
    src = torch.cat([lo, hi])
    dst = torch.cat([hi, lo])
    del lo, hi
    k2 = src * n + dst
    del src, dst
    k2, _ = torch.sort(k2)
    src = k2 // n
    cols = (k2 % n).to(torch.int32)
    del k2
    counts = torch.bincount(src, minlength=n)
    del src
    off = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    return off, cols


def erdos_renyi_pairs(n: int, avg_degree: float, seed: int, device="cpu"):
    """The raw sample multiset of erdos_renyi (loops and duplicates kept)."""
    m = int(n * avg_degree / 2)
    idx = torch.arange(m, dtype=torch.int64, device=device)
    return uniform_below(seed, idx, n, 1), uniform_below(seed, idx, n, 2)


def erdos_renyi(n: int, avg_degree: float, seed: int, device="cpu"):
    """n*avg_degree/2 uniform pairs, then dedup/loop removal (the
    oracle::random_graph recipe, tests/support/oracles.hpp:94-103)."""
    u, v = erdos_renyi_pairs(n, avg_degree, seed, device)
    return csr_from_edges(u, v, n)


def tri_mesh(nx: int, ny: int, seed: int, device="cpu"):
    """Triangulated grid: right, down and down-right diagonal edges
    (oracle::tri_grid shape, tests/support/oracles.hpp:119-130), ids permuted."""
    x = torch.arange(nx, dtype=torch.int64, device=device)
    y = torch.arange(ny, dtype=torch.int64, device=device)
    Y, X = torch.meshgrid(y, x, indexing="ij")
    X, Y = X.reshape(-1), Y.reshape(-1)
    ids = Y * nx + X
    us, vs = [], []
    for dx, dy in ((1, 0), (0, 1), (1, 1)):
        ok = (X + dx < nx) & (Y + dy < ny)
        us.append(ids[ok])
        vs.append(((Y + dy) * nx + (X + dx))[ok])
    u, v = torch.cat(us), torch.cat(vs)
    perm = random_permutation(nx * ny, seed, device)
    return csr_from_edges(perm[u], perm[v], nx * ny)


def stencil27(nx: int, ny: int, nz: int, seed: int, device="cpu"):
    """3D 27-point stencil: all 26 neighbours of the 3x3x3 cube, ids permuted."""
    n = nx * ny * nz
    ids = torch.arange(n, dtype=torch.int64, device=device)
    X = ids % nx
    Y = (ids // nx) % ny
    Z = ids // (nx * ny)
    us, vs = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if (dz, dy, dx) <= (0, 0, 0):
                    continue  # 13 forward directions; build symmetrises
                ok = ((X + dx >= 0) & (X + dx < nx) & (Y + dy >= 0) & (Y + dy < ny) &
                      (Z + dz >= 0) & (Z + dz < nz))
                us.append(ids[ok])
                vs.append(ids[ok] + dx + dy * nx + dz * nx * ny)
    u, v = torch.cat(us), torch.cat(vs)
    del us, vs
    perm = random_permutation(n, seed, device)
    return csr_from_edges(perm[u], perm[v], n)


def _rmat_samples(scale: int, a: float, b: float, c: float, seed: int, s0: int, s1: int, device):
    """Samples s0..s1-1 of the quadrant descent (one uniform draw per level)."""
    ab, abc = a + b, a + b + c
    idx = torch.arange(s0, s1, dtype=torch.int64, device=device)
    u = torch.zeros_like(idx)
    v = torch.zeros_like(idx)
    for level in range(scale):
        r = uniform01(seed, idx * scale + level, 3)
        u = (u << 1) | (r >= ab).to(torch.int64)
        v = (v << 1) | (((r >= a) & (r < ab)) | (r >= abc)).to(torch.int64)
    return u, v


def rmat_pairs(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int,
               device="cpu"):
    """The raw, relabelled sample multiset of rmat (loops and duplicates
    kept): what build_graph (graph.hpp:98-138) canonicalises."""
    n = 1 << scale
    perm = random_permutation(n, seed, device)
    u, v = _rmat_samples(scale, a, b, c, seed, 0, edge_factor * n, device)
    return perm[u], perm[v]


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int, device="cpu",
         chunk: int = 1 << 26, lean: bool = None):
    """R-MAT by recursive quadrant descent (generate_rmat, rmat.hpp:82-117):
    edge_factor * 2^scale samples, one uniform draw per level, then
    symmetrise/dedup/drop loops; ids randomly permuted (shuffle_vertices).
    Above 2^28 samples (scale 27: 2^31 samples, ~4.3 G directed entries) the
    bucketed builder keeps the peak memory near 4x the adjacency."""
    n = 1 << scale
    samples = edge_factor * n
    if lean is None:
        lean = samples > (1 << 28)
    perm = random_permutation(n, seed, device)
    if lean:
        return _rmat_csr_bucketed(scale, samples, a, b, c, seed, perm, device, chunk)
    us, vs = [], []
    for s0 in range(0, samples, chunk):
        u, v = _rmat_samples(scale, a, b, c, seed, s0, min(samples, s0 + chunk), device)
        us.append(u)
        vs.append(v)
    u, v = torch.cat(us), torch.cat(vs)
    del us, vs
    return csr_from_edges(perm[u], perm[v], n)


def _rmat_csr_bucketed(scale, samples, a, b, c, seed, perm, device, chunk, nbuckets=None):
    """The same canonical CSR as csr_from_edges(perm[u], perm[v]) without
    materialising the edge list several times: directed keys src*n + dst
    (both directions of every non-loop sample) are counted, then scattered,
    per bucket of source ids (two passes over the counter-based samples),
    and each bucket is sorted and deduplicated on its own.  Deduplicating
    directed keys is deduplicating undirected pairs, since every pair
    contributes both of its directions."""
    n = 1 << scale
    if nbuckets is None:
        nbuckets = 64 if scale >= 20 else 4
    shift = max(scale - (nbuckets.bit_length() - 1), 0)

    def directed(s0, s1):
        u, v = _rmat_samples(scale, a, b, c, seed, s0, s1, device)
        u, v = perm[u], perm[v]
        keep = u != v
        u, v = u[keep], v[keep]
        src = torch.cat([u, v])
        dst = torch.cat([v, u])
        return src, dst

    counts = torch.zeros(nbuckets, dtype=torch.int64, device=device)
    for s0 in range(0, samples, chunk):
        src, _ = directed(s0, min(samples, s0 + chunk))
        counts += torch.bincount(src >> shift, minlength=nbuckets)
    starts = torch.zeros(nbuckets + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=starts[1:])
    keys = torch.empty(int(starts[-1]), dtype=torch.int64, device=device)
    cursor = starts[:-1].clone()
    for s0 in range(0, samples, chunk):
        src, dst = directed(s0, min(samples, s0 + chunk))
        bkt = src >> shift
        order = torch.argsort(bkt, stable=True)
        k = (src * n + dst)[order]
        bc = torch.bincount(bkt, minlength=nbuckets)
        pos = torch.zeros(nbuckets + 1, dtype=torch.int64, device=device)
        torch.cumsum(bc, 0, out=pos[1:])
        for j, (p0, p1, cur) in enumerate(zip(pos[:-1].tolist(), pos[1:].tolist(), cursor.tolist())):
            if p1 > p0:
                keys[cur:cur + p1 - p0] = k[p0:p1]
        cursor += bc
        del src, dst, bkt, order, k
    deg = torch.zeros(n, dtype=torch.int64, device=device)
    col_parts = []
    total = 0
    for j in range(nbuckets):
        kb = keys[int(starts[j]):int(starts[j + 1])]
        if kb.numel() == 0:
            continue
        kb = torch.unique_consecutive(torch.sort(kb).values)
        deg += torch.bincount(kb // n, minlength=n)
        col_parts.append((kb % n).to(torch.int32))
        total += kb.numel()
    del keys
    cols = torch.empty(total, dtype=torch.int32, device=device)
    o = 0
    for part in col_parts:
        cols[o:o + part.numel()] = part
        o += part.numel()
    del col_parts
    off = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(deg, 0, out=off[1:])
    return off, cols


@dataclass(frozen=True)
class Config:
    name: str
    description: str
    index: int  # position in BASELINE.json configs


CONFIGS = {
    "er": Config("er", "Erdos-Renyi G(n=1,000,000, avg degree 16), ids random", 0),
    "tri": Config("tri", "2D triangular mesh 2000x2000 (deg ~6), ids permuted", 1),
    "stencil": Config("stencil", "3D 27-point stencil 200^3 (deg <= 26), ids permuted", 2),
    "rmat24": Config("rmat24", "R-MAT scale 24, ef 16, (.57,.19,.19,.05), ids permuted", 3),
    "rmat27": Config("rmat27", "R-MAT scale 27, ef 16, (.57,.19,.19,.05), ids permuted", 4),
}


def make_config(name: str, device="cuda", seed: int = 1, scale_down: int = 0):
    """The BASELINE.json configuration `name` (scale_down > 0 shrinks it for
    tests: halves linear sizes / subtracts from the R-MAT scale)."""
    if name == "er":
        return erdos_renyi(1_000_000 >> scale_down, 16.0, seed, device)
    if name == "tri":
        s = 2000 >> scale_down
        return tri_mesh(s, s, seed, device)
    if name == "stencil":
        s = 200 >> scale_down
        return stencil27(s, s, s, seed, device)
    if name == "rmat24":
        return rmat(24 - scale_down, 16, 0.57, 0.19, 0.19, seed, device)
    if name == "rmat27":
        return rmat(27 - scale_down, 16, 0.57, 0.19, 0.19, seed, device)
    raise ValueError(f"unknown config {name!r}")

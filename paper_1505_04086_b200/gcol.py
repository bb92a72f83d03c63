"""Host-side mirror of the reference `gcol` coloring interface, B200-backed.

Same names, argument meaning and error behaviour as the reference's
header-only C++ API (/root/reference/proj/include/gcol/), so code and tests
written against the reference read the same here:

    reference (C++)                         here
    ------------------------------------    -----------------------------------
    gcol::Graph, build_graph  graph.hpp     Graph, build_graph (host CSR; the
                                            device copy is made once, lazily)
    gcol::color_rsoc          parallel.hpp  color_rsoc      -> libgcol_cuda.so
    gcol::run_coloring        bench.hpp     run_coloring    -> libgcol_cuda.so
    gcol::first_fit_sequential coloring.hpp first_fit_sequential (device)
    gcol::detect_conflicts    coloring.hpp  detect_conflicts (device)
    gcol::verify_coloring     coloring.hpp  verify_coloring (device)
    gcol::count_colors        coloring.hpp  count_colors (device)
    ColoringStats/ColoringRun/ParallelOptions/Algorithm   same names
    input_error/capacity_error/verification_error         same names

Every coloring computation runs in the CUDA library; this module only builds
host CSR arrays (build_graph is host logic, as in the reference) and moves
buffers.  Without a CUDA device the calls raise NoDeviceError.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, List, NamedTuple, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import LIB

kUncolored = -1
kNoVertex = 0xFFFFFFFF


# --- errors (errors.hpp:11-52) ------------------------------------------------
class input_error(ValueError):
    """Semantically invalid arguments (errors.hpp:11)."""


class capacity_error(RuntimeError):
    """A size does not fit the index types in use (errors.hpp:37)."""


class verification_error(RuntimeError):
    """A run produced an improper or incomplete coloring (errors.hpp:43)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside libgcol_cuda."""


class NoDeviceError(RuntimeError):
    """No CUDA device: there is no CPU fallback."""


class RoundCapError(RuntimeError):
    """round_cap reached (the reference's sequential repair is not available)."""


_ERRORS = {
    _lib.GCOL_ERR_INVALID_ARGUMENT: input_error,
    _lib.GCOL_ERR_CAPACITY: capacity_error,
    _lib.GCOL_ERR_CUDA: CudaError,
    _lib.GCOL_ERR_NCCL: CudaError,
    _lib.GCOL_ERR_ROUND_CAP: RoundCapError,
    _lib.GCOL_ERR_VERIFY: verification_error,
    _lib.GCOL_ERR_NO_DEVICE: NoDeviceError,
}


def _check(rc: int) -> None:
    if rc != _lib.GCOL_OK:
        raise _ERRORS.get(rc, CudaError)(_lib.last_error() or f"gcol_cuda status {rc}")


# --- algorithm names (parallel.hpp:21-37) --------------------------------------
class Algorithm(enum.IntEnum):
    seq = _lib.ALG_SEQ
    catalyurek = _lib.ALG_CATALYUREK
    rsoc = _lib.ALG_RSOC


def to_string(a: Algorithm) -> str:
    return Algorithm(a).name


def algorithm_from_string(name: str) -> Optional[Algorithm]:
    return Algorithm[name] if name in Algorithm.__members__ else None


class Priority(enum.IntEnum):
    """Which endpoint of a monochromatic edge recolors (include/gcol_cuda.h)."""
    id_low = _lib.PRIORITY_ID_LOW        # reference rule, coloring.hpp:118-120
    id_high = _lib.PRIORITY_ID_HIGH
    degree_id = _lib.PRIORITY_DEGREE_ID
    ordered = _lib.PRIORITY_ORDERED      # north_star rule; converges towards serial FF


@dataclass
class ParallelOptions:
    """parallel.hpp:64-72 plus the device knobs of gcol_cuda_options."""
    chunk_size: int = 0
    min_chunk_size: int = 64
    round_cap: int = 1000
    priority: Priority = Priority.degree_id  # library default
    k1_blocks_per_sm: int = 0
    k1_read_all: bool = False
    k1_split_min_degree: int = 0
    k1_wide: int = 0
    k1_wait_polls: int = 0

    def to_c(self, thread_count: int) -> _lib.Options:
        o = _lib.Options()
        o.struct_size = C.sizeof(_lib.Options)
        o.thread_count = thread_count
        o.chunk_size = self.chunk_size
        o.min_chunk_size = self.min_chunk_size
        o.round_cap = self.round_cap
        o.priority = int(self.priority)
        o.k1_blocks_per_sm = self.k1_blocks_per_sm
        o.k1_read_all = 1 if self.k1_read_all else 0
        o.k1_split_min_degree = self.k1_split_min_degree
        o.k1_wide = self.k1_wide
        o.k1_wait_polls = self.k1_wait_polls
        return o


@dataclass
class ColoringStats:
    """parallel.hpp:47-57 (+ device instrumentation)."""
    algorithm: Algorithm = Algorithm.seq
    thread_count: int = 1
    rounds: int = 0
    conflicts_total: int = 0
    conflicts_per_round: List[int] = field(default_factory=list)
    barrier_events: int = 0
    num_colors: int = 0
    wall_time_ns: int = 0
    fallback_triggered: bool = False
    initial_pass_ns: int = 0
    pairs_logged: int = 0
    round1_candidates: int = 0
    pair_overflow: bool = False
    priority: Priority = Priority.degree_id
    k1_gathers: int = 0
    h2d_bytes: int = 0       # bytes the call copied host -> device (incl. the upload
    d2h_bytes: int = 0       # on a handle's first call) / device -> host
    heavy_pass_ns: int = 0   # class-split initial pass: device time of the heavy-row pass
    heavy_rows: int = 0      # rows of that pass (degree >= 64); 0 when not split


@dataclass
class ColoringRun:
    coloring: np.ndarray
    stats: ColoringStats


class Violation(NamedTuple):
    u: int
    v: int
    color: int


@dataclass
class ConflictReport:
    """coloring.hpp:146-157."""
    violations: List[Violation]

    def ok(self) -> bool:
        return not self.violations


# --- Graph (graph.hpp:20-93) ---------------------------------------------------
class Graph:
    """Immutable undirected CSR graph: int64 offsets (n+1), int32 neighbours
    (2|E|), rows sorted ascending, symmetric, no self-loops or duplicates.
    The device copy is created on first use and reused (the reference's
    Graph is shared read-only across runs the same way)."""

    def __init__(self, offsets: np.ndarray, adjacency: np.ndarray, *, _max_degree=None,
                 _device_arrays=None):
        self._off = np.ascontiguousarray(offsets, dtype=np.int64)
        self._adj = np.ascontiguousarray(adjacency, dtype=np.int32)
        if self._off.ndim != 1 or self._off.size < 1:
            raise input_error("graph: offsets array has wrong length")
        n = self._off.size - 1
        if n >= 2 ** 31 - 1:
            raise capacity_error("vertex count exceeds the 31-bit id space")
        if _max_degree is None:
            _max_degree = int(np.diff(self._off).max()) if n > 0 else 0
        self._maxdeg = int(_max_degree)
        self._m = int(self._off[-1])
        self._handle = None
        self._device_arrays = _device_arrays  # (torch offsets, torch cols) when device-resident

    # graph.hpp:24-45
    def num_vertices(self) -> int:
        return self._off.size - 1

    def num_edges(self) -> int:
        return self._m // 2

    def num_adjacency(self) -> int:
        """m = 2|E| directed adjacency entries."""
        return self._m

    def max_degree(self) -> int:
        return self._maxdeg

    def _check_vertex(self, v: int) -> None:
        if not 0 <= v < self.num_vertices():
            raise input_error(f"vertex id {v} out of range (|V| = {self.num_vertices()})")

    def degree(self, v: int) -> int:
        self._check_vertex(v)
        return int(self._off[v + 1] - self._off[v])

    def neighbors(self, v: int) -> np.ndarray:
        self._check_vertex(v)
        return self._adj[self._off[v]:self._off[v + 1]]

    def offsets(self) -> np.ndarray:
        return self._off

    def adjacency(self) -> np.ndarray:
        return self._adj

    def __eq__(self, other) -> bool:
        return (isinstance(other, Graph) and np.array_equal(self._off, other._off)
                and np.array_equal(self._adj, other._adj))

    def validate(self) -> None:
        """graph.hpp:50-77: every structural invariant, input_error on violation."""
        off, adj = self._off, self._adj
        n = self.num_vertices()
        if off[0] != 0 or off[-1] != adj.size:
            raise input_error("graph: offsets do not cover the adjacency array")
        deg = np.diff(off)
        if (deg < 0).any():
            raise input_error("graph: offsets are not monotone")
        if adj.size:
            if adj.min() < 0 or adj.max() >= n:
                raise input_error("graph: neighbor id out of range")
            rows = np.repeat(np.arange(n, dtype=np.int64), deg)
            if (adj == rows).any():
                raise input_error("graph: self-loop present")
            same_row = rows[1:] == rows[:-1]
            if (same_row & (adj[1:] <= adj[:-1])).any():
                raise input_error("graph: adjacency list not sorted strictly ascending")
            fwd = rows * n + adj
            bwd = adj.astype(np.int64) * n + rows
            if not np.array_equal(np.sort(fwd), np.sort(bwd)):
                raise input_error("graph: edge stored in one direction only")
        if (int(deg.max()) if n else 0) != self._maxdeg:
            raise input_error("graph: cached max degree is stale")

    # -- device handle --------------------------------------------------------
    def handle(self) -> C.c_void_p:
        if self._handle is None:
            h = C.c_void_p()
            if self._device_arrays is not None:
                d_off, d_cols = self._device_arrays
                _check(LIB.gcol_cuda_graph_create(
                    C.c_void_p(d_off.data_ptr()), C.c_void_p(d_cols.data_ptr()),
                    self.num_vertices(), self._m, _lib.GCOL_MEM_DEVICE,
                    d_off.device.index if d_off.device.index is not None else -1, C.byref(h)))
            else:
                _check(LIB.gcol_cuda_graph_create(
                    self._off.ctypes.data_as(C.c_void_p), self._adj.ctypes.data_as(C.c_void_p),
                    self.num_vertices(), self._adj.size, _lib.GCOL_MEM_HOST, -1, C.byref(h)))
            self._handle = h
        return self._handle

    def release(self) -> None:
        if self._handle is not None:
            LIB.gcol_cuda_graph_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    @classmethod
    def from_device(cls, d_offsets, d_cols, host_offsets: Optional[np.ndarray] = None,
                    max_degree: Optional[int] = None) -> "Graph":
        """Wrap a CSR already resident in HBM (torch CUDA tensors, int64 /
        int32).  Host arrays are not required for coloring; offsets are
        copied back only if not supplied (for degree queries)."""
        if host_offsets is None:
            host_offsets = d_offsets.cpu().numpy()
        return cls(host_offsets, np.empty(0, np.int32), _max_degree=max_degree,
                   _device_arrays=(d_offsets, d_cols))


def build_graph(edges, num_vertices: int) -> Graph:
    """graph.hpp:98-138: canonical CSR from an unordered edge list.  Self-loops
    dropped, duplicates in either orientation collapsed, ids must be
    < num_vertices (input_error otherwise).  Host logic (numpy)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2) if len(edges) else np.zeros((0, 2), np.int64)
    n = int(num_vertices)
    if n < 0:
        raise input_error("num_vertices must be non-negative")
    if e.size and (e.min() < 0 or e.max() >= n):
        bad = e[(e < 0).any(axis=1) | (e >= n).any(axis=1)][0]
        raise input_error(f"edge ({bad[0]}, {bad[1]}) references a vertex id >= {n}")
    e = e[e[:, 0] != e[:, 1]]
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    key = np.unique(lo * max(n, 1) + hi)
    lo, hi = key // max(n, 1), key % max(n, 1)
    src = np.concatenate([lo, hi])
    dst = np.concatenate([hi, lo])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    counts = np.bincount(src, minlength=n) if n else np.zeros(0, np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return Graph(off, dst.astype(np.int32))


# --- buffers ---------------------------------------------------------------------
def _as_host_i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


def _stats_from_c(s: _lib.Stats, cpr: np.ndarray) -> ColoringStats:
    return ColoringStats(
        algorithm=Algorithm(s.algorithm), thread_count=s.thread_count, rounds=s.rounds,
        conflicts_total=s.conflicts_total,
        conflicts_per_round=[int(x) for x in cpr[:min(s.cpr_len, cpr.size)]],
        barrier_events=s.barrier_events, num_colors=s.num_colors,
        wall_time_ns=s.wall_time_ns, fallback_triggered=bool(s.fallback_triggered),
        initial_pass_ns=s.initial_pass_ns, pairs_logged=s.pairs_logged,
        round1_candidates=s.round1_candidates, pair_overflow=bool(s.pair_overflow),
        priority=Priority(s.priority), k1_gathers=s.k1_gathers, h2d_bytes=s.h2d_bytes,
        d2h_bytes=s.d2h_bytes, heavy_pass_ns=s.heavy_pass_ns, heavy_rows=s.heavy_rows)


# --- coloring entry points -------------------------------------------------------
def run_coloring(g: Graph, algorithm: Algorithm, thread_count: int,
                 opt: Optional[ParallelOptions] = None, *, colors_out=None) -> ColoringRun:
    """bench.hpp:35-60 on the device.  colors_out: optional preallocated
    output (numpy int32 host array or torch int32 CUDA tensor)."""
    if thread_count < 1:
        raise input_error("thread_count must be at least 1")
    opt = opt or ParallelOptions()
    n = g.num_vertices()
    cap = max(int(opt.round_cap), 1) + 1
    cpr = np.zeros(min(cap, 1 << 16), dtype=np.uint64)
    st = _lib.Stats()
    st.conflicts_per_round = cpr.ctypes.data_as(C.POINTER(C.c_uint64))
    st.cpr_cap = cpr.size
    copt = opt.to_c(thread_count)
    if colors_out is None:
        out = np.empty(n, dtype=np.int32)
        optr, mem = _ptr(out), _lib.GCOL_MEM_HOST
    elif isinstance(colors_out, np.ndarray):
        out = colors_out
        optr, mem = _ptr(out), _lib.GCOL_MEM_HOST
    else:  # torch CUDA tensor
        out = colors_out
        optr, mem = C.c_void_p(out.data_ptr()), _lib.GCOL_MEM_DEVICE
    _check(LIB.gcol_cuda_run_coloring(g.handle(), int(algorithm), C.byref(copt), optr, mem,
                                      C.byref(st)))
    return ColoringRun(out, _stats_from_c(st, cpr))


def color_rsoc(g: Graph, thread_count: int, opt: Optional[ParallelOptions] = None,
               **kw) -> ColoringRun:
    """parallel.hpp:253-319 on the device (fused detect-and-recolor rounds)."""
    return run_coloring(g, Algorithm.rsoc, thread_count, opt, **kw)


def color_catalyurek(g: Graph, thread_count: int, opt: Optional[ParallelOptions] = None,
                     **kw) -> ColoringRun:
    """parallel.hpp:180-246 on the device (tentative phase, then detection)."""
    return run_coloring(g, Algorithm.catalyurek, thread_count, opt, **kw)


def color_rsoc_csr(offsets, adjacency, thread_count: int,
                   opt: Optional[ParallelOptions] = None, *, colors_out=None,
                   device: int = -1) -> ColoringRun:
    """color_rsoc on a host CSR in one call (parallel.hpp:253 with a host
    Graph): the adjacency upload is overlapped with the initial pass
    (gcol_cuda_color_rsoc_csr).  offsets/adjacency: int64 / int32 host arrays
    (numpy, or CPU torch tensors -- pinned ones upload asynchronously);
    colors_out: optional int32 host array of n entries."""
    if thread_count < 1:
        raise input_error("thread_count must be at least 1")
    opt = opt or ParallelOptions()

    def host_ptr(a, dtype):
        if isinstance(a, np.ndarray):
            a = np.ascontiguousarray(a, dtype=dtype)
            return a, _ptr(a), a.size
        if a.is_cuda:
            raise input_error("color_rsoc_csr takes host arrays")
        return a, C.c_void_p(a.data_ptr()), a.numel()

    off_keep, off_p, n1 = host_ptr(offsets, np.int64)
    cols_keep, cols_p, m = host_ptr(adjacency, np.int32)
    n = n1 - 1
    if n < 0:
        raise input_error("offsets must hold n + 1 entries")
    cap = max(int(opt.round_cap), 1) + 1
    cpr = np.zeros(min(cap, 1 << 16), dtype=np.uint64)
    st = _lib.Stats()
    st.conflicts_per_round = cpr.ctypes.data_as(C.POINTER(C.c_uint64))
    st.cpr_cap = cpr.size
    copt = opt.to_c(thread_count)
    if colors_out is None:
        out = np.empty(n, dtype=np.int32)
        optr = _ptr(out)
    elif isinstance(colors_out, np.ndarray):
        out = colors_out
        optr = _ptr(out)
    else:  # CPU torch tensor (e.g. pinned)
        out = colors_out
        optr = C.c_void_p(out.data_ptr())
    _check(LIB.gcol_cuda_color_rsoc_csr(off_p, cols_p, n, m, int(device), C.byref(copt), optr,
                                        C.byref(st)))
    del off_keep, cols_keep
    return ColoringRun(out, _stats_from_c(st, cpr))


def first_fit_sequential(g: Graph) -> np.ndarray:
    """coloring.hpp:110-116 on the device; bit-identical to the reference."""
    out = np.empty(g.num_vertices(), dtype=np.int32)
    _check(LIB.gcol_cuda_first_fit_sequential(g.handle(), _ptr(out), _lib.GCOL_MEM_HOST))
    return out


def tentative_snapshot(g: Graph, colors_in, worklist: Optional[Sequence[int]] = None,
                       lower_only: bool = False) -> np.ndarray:
    """K1 in snapshot mode: smallest_available_color (coloring.hpp:95-106) of
    each worklist vertex over the frozen colors_in; others keep colors_in."""
    cin = _as_host_i32(colors_in)
    if cin.size != g.num_vertices():
        raise input_error("coloring size does not match graph")
    out = np.empty_like(cin)
    if worklist is None:
        _check(LIB.gcol_cuda_tentative_snapshot(g.handle(), _ptr(cin), None, 0,
                                                1 if lower_only else 0, _ptr(out),
                                                _lib.GCOL_MEM_HOST))
    else:
        wl = _as_host_i32(worklist)
        _check(LIB.gcol_cuda_tentative_snapshot(g.handle(), _ptr(cin), _ptr(wl), wl.size,
                                                1 if lower_only else 0, _ptr(out),
                                                _lib.GCOL_MEM_HOST))
    return out


def detect_conflicts(g: Graph, coloring, pending: Iterable[int],
                     priority: Priority = Priority.id_low) -> List[int]:
    """coloring.hpp:133-141: the defective subset of `pending`, in order."""
    c = _as_host_i32(coloring)
    if c.size != g.num_vertices():
        raise input_error("detect_conflicts: coloring size does not match graph")
    wl = _as_host_i32(list(pending))
    flags = np.zeros(wl.size, dtype=np.int32)
    if wl.size:
        _check(LIB.gcol_cuda_detect_conflicts(g.handle(), _ptr(c), _ptr(wl), wl.size,
                                              int(priority), _ptr(flags), _lib.GCOL_MEM_HOST))
    return [int(v) for v, f in zip(wl, flags) if f]


def detect_and_recolor(g: Graph, coloring, pending: Iterable[int],
                       priority: Priority = Priority.id_low) -> Tuple[np.ndarray, List[int]]:
    """One fused RSOC round body (parallel.hpp:297-313) over `pending`:
    returns (new colours, recoloured ids).  Deterministic for independent sets."""
    c = _as_host_i32(coloring).copy()
    if c.size != g.num_vertices():
        raise input_error("coloring size does not match graph")
    wl = _as_host_i32(list(pending))
    out = np.zeros(max(wl.size, 1), dtype=np.int32)
    nout = C.c_int64(0)
    if wl.size:
        _check(LIB.gcol_cuda_detect_and_recolor(g.handle(), _ptr(c), _ptr(wl), wl.size,
                                                int(priority), _ptr(out), C.byref(nout),
                                                _lib.GCOL_MEM_HOST))
    return c, sorted(int(x) for x in out[:nout.value])


def verify_report(g: Graph, coloring, cap: int = 0):
    c = _as_host_i32(coloring)
    rep = _lib.VerifyReport()
    u = np.zeros(max(cap, 1), dtype=np.uint32)
    v = np.zeros(max(cap, 1), dtype=np.uint32)
    col = np.zeros(max(cap, 1), dtype=np.int32)
    _check(LIB.gcol_cuda_verify_coloring(g.handle(), _ptr(c), c.size, _lib.GCOL_MEM_HOST,
                                         C.byref(rep), _ptr(u), _ptr(v), _ptr(col), cap))
    return rep, u, v, col


def verify_coloring(g: Graph, coloring) -> ConflictReport:
    """coloring.hpp:159-177: every violation, in the reference order."""
    c = _as_host_i32(coloring)
    if c.size != g.num_vertices():
        raise input_error(f"verify_coloring: coloring has {c.size} entries, graph has "
                          f"{g.num_vertices()} vertices")
    rep, _, _, _ = verify_report(g, c, 0)
    cap = int(rep.violations)
    if cap == 0:
        return ConflictReport([])
    rep, u, v, col = verify_report(g, c, cap)
    return ConflictReport([Violation(int(a), int(b), int(x)) for a, b, x in zip(u, v, col)])


def count_colors(coloring, g: Optional[Graph] = None) -> int:
    """coloring.hpp:181-196: number of DISTINCT colours (device census).
    Incomplete or negative colourings raise input_error."""
    c = _as_host_i32(coloring)
    if g is None or g.num_vertices() != c.size:
        g = Graph(np.zeros(c.size + 1, np.int64), np.zeros(0, np.int32), _max_degree=0)
    out = C.c_uint32(0)
    _check(LIB.gcol_cuda_count_colors(g.handle(), _ptr(c), c.size, _lib.GCOL_MEM_HOST,
                                      C.byref(out)))
    return int(out.value)


def device_count() -> int:
    n = C.c_int32(0)
    LIB.gcol_cuda_device_count(C.byref(n))
    return int(n.value)

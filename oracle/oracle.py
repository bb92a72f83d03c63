"""ctypes bindings of the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs (see gcol_oracle.h).  Two libraries:

  oracle/libgcol_oracle.so   our C restatement (gcol_oracle.c), always built
  oracle/_ref/libgcolref.so  the reference's own header-only library compiled
                             from /root/reference (ref_wrapper.cpp); optional
                             on machines where it was not built
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libgcol_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgcolref.so")


class OracleStats(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32),
        ("thread_count", C.c_uint32),
        ("rounds", C.c_uint64),
        ("conflicts_total", C.c_uint64),
        ("barrier_events", C.c_uint64),
        ("num_colors", C.c_uint32),
        ("fallback_triggered", C.c_uint32),
        ("wall_time_ns", C.c_uint64),
        ("cpr_len", C.c_uint64),
        ("conflicts_per_round", C.POINTER(C.c_uint64)),
        ("cpr_cap", C.c_uint64),
    ]


def build(quiet: bool = True) -> None:
    """make -C oracle (C restatement + reference shim when headers exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _load(path: str) -> C.CDLL:
    return C.CDLL(path)


_vp = C.c_void_p
_oracle: Optional[C.CDLL] = None
_ref: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = _load(ORACLE_SO)
        L.oracle_build_graph.restype = C.c_int64
        L.oracle_build_graph.argtypes = [_vp, C.c_int64, C.c_uint32, _vp, _vp, C.c_int64, _vp]
        L.oracle_smallest_available_color.restype = C.c_int32
        L.oracle_smallest_available_color.argtypes = [_vp, _vp, _vp, C.c_uint32]
        L.oracle_tentative_snapshot.restype = None
        L.oracle_tentative_snapshot.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, _vp]
        L.oracle_first_fit_sequential.restype = None
        L.oracle_first_fit_sequential.argtypes = [_vp, _vp, C.c_uint32, _vp]
        L.oracle_has_conflicting_higher_neighbor.restype = C.c_int
        L.oracle_has_conflicting_higher_neighbor.argtypes = [_vp, _vp, _vp, C.c_uint32]
        L.oracle_detect_conflicts.restype = C.c_int64
        L.oracle_detect_conflicts.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, _vp]
        L.oracle_verify_coloring.restype = C.c_int64
        L.oracle_verify_coloring.argtypes = [_vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp, C.c_int64]
        L.oracle_count_colors.restype = C.c_int64
        L.oracle_count_colors.argtypes = [_vp, C.c_int64]
        for name in ("oracle_color_rsoc", "oracle_color_catalyurek"):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = [_vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                           C.c_uint64, _vp, C.POINTER(OracleStats)]
        L.oracle_lockstep_color.restype = C.c_int64
        L.oracle_lockstep_color.argtypes = [_vp, _vp, C.c_uint32, _vp, C.c_uint64, _vp, _vp]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = _load(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_graph.restype = _vp
        L.ref_build_graph.argtypes = [_vp, C.c_int64, C.c_uint32, C.POINTER(C.c_int)]
        L.ref_graph_from_csr.restype = _vp
        L.ref_graph_from_csr.argtypes = [_vp, _vp, C.c_uint32, C.POINTER(C.c_int)]
        L.ref_graph_free.argtypes = [_vp]
        L.ref_num_vertices.restype = C.c_uint32
        L.ref_num_vertices.argtypes = [_vp]
        L.ref_num_adjacency.restype = C.c_uint64
        L.ref_num_adjacency.argtypes = [_vp]
        L.ref_max_degree.restype = C.c_uint32
        L.ref_max_degree.argtypes = [_vp]
        L.ref_graph_csr.argtypes = [_vp, _vp, _vp]
        L.ref_color.restype = C.c_int
        L.ref_color.argtypes = [_vp, C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, _vp,
                                C.POINTER(OracleStats)]
        L.ref_smallest_available_color.restype = C.c_int32
        L.ref_smallest_available_color.argtypes = [_vp, _vp, C.c_uint32]
        L.ref_detect_conflicts.restype = C.c_int64
        L.ref_detect_conflicts.argtypes = [_vp, _vp, C.c_int64, _vp, C.c_int64, _vp]
        L.ref_verify_coloring.restype = C.c_int64
        L.ref_verify_coloring.argtypes = [_vp, _vp, C.c_int64, _vp, _vp, _vp, C.c_int64]
        L.ref_count_colors.restype = C.c_int64
        L.ref_count_colors.argtypes = [_vp, C.c_int64]
        L.ref_first_fit_sequential.restype = C.c_int
        L.ref_first_fit_sequential.argtypes = [_vp, _vp]
        L.ref_lockstep_color.restype = C.c_int64
        L.ref_lockstep_color.argtypes = [_vp, _vp, C.c_int64, C.c_uint64, _vp, _vp]
        L.ref_generate_rmat.restype = _vp
        L.ref_generate_rmat.argtypes = [C.c_uint, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_shuffle_vertices.restype = _vp
        L.ref_shuffle_vertices.argtypes = [_vp, C.c_uint64, _vp]
        L.ref_parse_text.restype = _vp
        L.ref_parse_text.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int64, C.POINTER(C.c_int),
                                     C.POINTER(C.c_uint64)]
        L.ref_save_edge_list.restype = C.c_uint64
        L.ref_save_edge_list.argtypes = [_vp, C.c_char_p, C.c_uint64]
        _ref = L
    return _ref


def _p(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------
class CSR:
    """Canonical CSR as the oracle sees it (uint64 offsets, uint32 cols)."""

    def __init__(self, off: np.ndarray, cols: np.ndarray, max_degree: Optional[int] = None):
        self.off = np.ascontiguousarray(off, dtype=np.uint64)
        self.cols = np.ascontiguousarray(cols, dtype=np.uint32)
        self.n = self.off.size - 1
        if max_degree is None:
            max_degree = int(np.diff(self.off.astype(np.int64)).max()) if self.n else 0
        self.max_degree = max_degree


def build_graph(edges, n: int) -> CSR:
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
    off = np.zeros(n + 1, dtype=np.uint64)
    cols = np.zeros(max(2 * len(e), 1), dtype=np.uint32)
    md = C.c_uint32(0)
    m = lib().oracle_build_graph(_p(e), len(e), n, _p(off), _p(cols), cols.size, C.byref(md))
    if m == -1:
        raise ValueError("edge references a vertex id >= num_vertices")
    return CSR(off, cols[:m].copy(), md.value)


def smallest_available_color(g: CSR, colors, v: int) -> int:
    c = np.ascontiguousarray(colors, dtype=np.int32)
    return lib().oracle_smallest_available_color(_p(g.off), _p(g.cols), _p(c), v)


def tentative_snapshot(g: CSR, colors_in, worklist=None, lower_only: bool = False) -> np.ndarray:
    cin = np.ascontiguousarray(colors_in, dtype=np.int32)
    wl = np.arange(g.n, dtype=np.uint32) if worklist is None else \
        np.ascontiguousarray(worklist, dtype=np.uint32)
    out = cin.copy()
    if not lower_only:
        lib().oracle_tentative_snapshot(_p(g.off), _p(g.cols), _p(cin), _p(wl), wl.size, _p(out))
        return out
    # lower-only variant: First-Fit over the neighbours with id < v (the
    # initial-pass neighbourhood of an ascending sweep)
    for v in wl:
        b, e = int(g.off[v]), int(g.off[v + 1])
        nb = g.cols[b:e]
        nb = nb[nb < v]
        used = set(int(x) for x in cin[nb] if 0 <= x <= e - b)
        c = 0
        while c in used:
            c += 1
        out[v] = c
    return out


def first_fit_sequential(g: CSR) -> np.ndarray:
    out = np.empty(g.n, dtype=np.int32)
    lib().oracle_first_fit_sequential(_p(g.off), _p(g.cols), g.n, _p(out))
    return out


def detect_conflicts(g: CSR, colors, pending) -> List[int]:
    c = np.ascontiguousarray(colors, dtype=np.int32)
    p = np.ascontiguousarray(pending, dtype=np.uint32)
    out = np.zeros(max(p.size, 1), dtype=np.uint32)
    k = lib().oracle_detect_conflicts(_p(g.off), _p(g.cols), _p(c), _p(p), p.size, _p(out))
    return [int(x) for x in out[:k]]


def verify_coloring(g: CSR, colors) -> List[Tuple[int, int, int]]:
    c = np.ascontiguousarray(colors, dtype=np.int32)
    k = lib().oracle_verify_coloring(_p(g.off), _p(g.cols), g.n, _p(c), None, None, None, 0)
    u = np.zeros(max(k, 1), np.uint32)
    v = np.zeros(max(k, 1), np.uint32)
    cc = np.zeros(max(k, 1), np.int32)
    lib().oracle_verify_coloring(_p(g.off), _p(g.cols), g.n, _p(c), _p(u), _p(v), _p(cc), k)
    return [(int(a), int(b), int(x)) for a, b, x in zip(u[:k], v[:k], cc[:k])]


def count_colors(colors) -> int:
    c = np.ascontiguousarray(colors, dtype=np.int32)
    return int(lib().oracle_count_colors(_p(c), c.size))


def _stats_dict(st: OracleStats, cpr: np.ndarray) -> Dict:
    return dict(algorithm=st.algorithm, thread_count=st.thread_count, rounds=st.rounds,
                conflicts_total=st.conflicts_total, barrier_events=st.barrier_events,
                num_colors=st.num_colors, fallback_triggered=bool(st.fallback_triggered),
                wall_time_ns=st.wall_time_ns,
                conflicts_per_round=[int(x) for x in cpr[:min(st.cpr_len, cpr.size)]])


def color_parallel(g: CSR, threads: int, algorithm: str = "rsoc", chunk_size: int = 0,
                   min_chunk_size: int = 64, round_cap: int = 1000):
    out = np.empty(max(g.n, 1), dtype=np.int32)
    cpr = np.zeros(4096, dtype=np.uint64)
    st = OracleStats()
    st.conflicts_per_round = cpr.ctypes.data_as(C.POINTER(C.c_uint64))
    st.cpr_cap = cpr.size
    fn = lib().oracle_color_rsoc if algorithm == "rsoc" else lib().oracle_color_catalyurek
    rc = fn(_p(g.off), _p(g.cols), g.n, g.max_degree, threads, chunk_size, min_chunk_size,
            round_cap, _p(out), C.byref(st))
    if rc == -1:
        raise ValueError("thread_count must be at least 1")
    if rc != 0:
        raise RuntimeError("parallel coloring finished improper")
    return out[:g.n], _stats_dict(st, cpr)


def lockstep_color(g: CSR, lanes, round_cap: int):
    lanes = np.ascontiguousarray(lanes, dtype=np.uint32)
    trace = np.zeros(max(round_cap * g.n, 1), dtype=np.int32)
    conv = C.c_int32(0)
    r = lib().oracle_lockstep_color(_p(g.off), _p(g.cols), g.n, _p(lanes), round_cap, _p(trace),
                                    C.byref(conv))
    if r < 0:
        raise ValueError("bad lockstep arguments")
    return bool(conv.value), int(r), trace[:r * g.n].reshape(r, g.n) if g.n else np.zeros((r, 0))


# ---------------------------------------------------------------------------
# The reference itself (oracle/_ref)
# ---------------------------------------------------------------------------
class RefGraph:
    """A gcol::Graph built by the reference's own build_graph."""

    def __init__(self, ptr):
        self.ptr = C.c_void_p(ptr)
        L = ref()
        self.n = L.ref_num_vertices(self.ptr)
        self.m = L.ref_num_adjacency(self.ptr)
        self.max_degree = L.ref_max_degree(self.ptr)

    @classmethod
    def from_edges(cls, edges, n: int) -> "RefGraph":
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        st = C.c_int(0)
        p = ref().ref_build_graph(_p(e), len(e), n, C.byref(st))
        if st.value != 0:
            raise ValueError(ref().ref_last_error().decode())
        return cls(p)

    @classmethod
    def from_csr(cls, off, cols) -> "RefGraph":
        off = np.ascontiguousarray(off, dtype=np.uint64)
        cols = np.ascontiguousarray(cols, dtype=np.uint32)
        st = C.c_int(0)
        p = ref().ref_graph_from_csr(_p(off), _p(cols), off.size - 1, C.byref(st))
        if st.value != 0:
            raise ValueError(ref().ref_last_error().decode())
        return cls(p)

    @classmethod
    def parse_text(cls, text: bytes, fmt: str = "edgelist", num_vertices: int = -1):
        """The reference's load_edge_list / load_matrix_market on `text`.
        Returns (graph, None) or (None, (kind, line, message))."""
        st, line = C.c_int(0), C.c_uint64(0)
        p = ref().ref_parse_text(text, len(text), 2 if fmt == "mm" else 1, num_vertices,
                                 C.byref(st), C.byref(line))
        if st.value != 0:
            kind = {-1: "input", -2: "capacity", -5: "parse", -6: "unsupported_format"}.get(st.value, "other")
            return None, (kind, int(line.value), ref().ref_last_error().decode())
        return cls(p), None

    def save_edge_list(self) -> bytes:
        k = ref().ref_save_edge_list(self.ptr, None, 0)
        buf = C.create_string_buffer(int(k) + 1)
        ref().ref_save_edge_list(self.ptr, buf, k)
        return buf.raw[:k]

    @classmethod
    def rmat(cls, scale, edge_factor, a, b, c, d, seed) -> "RefGraph":
        st = C.c_int(0)
        p = ref().ref_generate_rmat(scale, edge_factor, a, b, c, d, seed, C.byref(st))
        if st.value != 0:
            raise ValueError(ref().ref_last_error().decode())
        return cls(p)

    def shuffled(self, seed: int):
        perm = np.zeros(max(self.n, 1), dtype=np.uint32)
        p = ref().ref_shuffle_vertices(self.ptr, seed, _p(perm))
        return RefGraph(p), perm[:self.n]

    def csr(self) -> CSR:
        off = np.zeros(self.n + 1, dtype=np.uint64)
        cols = np.zeros(max(self.m, 1), dtype=np.uint32)
        ref().ref_graph_csr(self.ptr, _p(off), _p(cols))
        return CSR(off, cols[:self.m], self.max_degree)

    def color(self, algorithm: str, threads: int, chunk_size: int = 0, min_chunk_size: int = 64,
              round_cap: int = 1000):
        alg = {"seq": 0, "catalyurek": 1, "rsoc": 2}[algorithm]
        out = np.empty(max(self.n, 1), dtype=np.int32)
        cpr = np.zeros(4096, dtype=np.uint64)
        st = OracleStats()
        st.conflicts_per_round = cpr.ctypes.data_as(C.POINTER(C.c_uint64))
        st.cpr_cap = cpr.size
        rc = ref().ref_color(self.ptr, alg, threads, chunk_size, min_chunk_size, round_cap, _p(out),
                             C.byref(st))
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {ref().ref_last_error().decode()}")
        return out[:self.n], _stats_dict(st, cpr)

    def first_fit_sequential(self) -> np.ndarray:
        out = np.empty(max(self.n, 1), dtype=np.int32)
        ref().ref_first_fit_sequential(self.ptr, _p(out))
        return out[:self.n]

    def smallest_available_color(self, colors, v: int) -> int:
        c = np.ascontiguousarray(colors, dtype=np.int32)
        return ref().ref_smallest_available_color(self.ptr, _p(c), v)

    def detect_conflicts(self, colors, pending) -> List[int]:
        c = np.ascontiguousarray(colors, dtype=np.int32)
        p = np.ascontiguousarray(pending, dtype=np.uint32)
        out = np.zeros(max(p.size, 1), dtype=np.uint32)
        k = ref().ref_detect_conflicts(self.ptr, _p(c), c.size, _p(p), p.size, _p(out))
        if k < 0:
            raise ValueError(ref().ref_last_error().decode())
        return [int(x) for x in out[:k]]

    def verify_coloring(self, colors) -> List[Tuple[int, int, int]]:
        c = np.ascontiguousarray(colors, dtype=np.int32)
        k = ref().ref_verify_coloring(self.ptr, _p(c), c.size, None, None, None, 0)
        if k < 0:
            raise ValueError(ref().ref_last_error().decode())
        u = np.zeros(max(k, 1), np.uint32)
        v = np.zeros(max(k, 1), np.uint32)
        cc = np.zeros(max(k, 1), np.int32)
        ref().ref_verify_coloring(self.ptr, _p(c), c.size, _p(u), _p(v), _p(cc), k)
        return [(int(a), int(b), int(x)) for a, b, x in zip(u[:k], v[:k], cc[:k])]

    def lockstep_color(self, lanes, round_cap: int):
        lanes = np.ascontiguousarray(lanes, dtype=np.uint32)
        trace = np.zeros(max(round_cap * self.n, 1), dtype=np.int32)
        conv = C.c_int32(0)
        r = ref().ref_lockstep_color(self.ptr, _p(lanes), lanes.size, round_cap, _p(trace),
                                     C.byref(conv))
        if r < 0:
            raise ValueError(ref().ref_last_error().decode())
        return bool(conv.value), int(r), trace[:r * self.n].reshape(r, self.n) if self.n else \
            np.zeros((r, 0))

    def __del__(self):
        try:
            ref().ref_graph_free(self.ptr)
        except Exception:
            pass


def ref_count_colors(colors) -> int:
    c = np.ascontiguousarray(colors, dtype=np.int32)
    return int(ref().ref_count_colors(_p(c), c.size))

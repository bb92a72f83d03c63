"""Text ingestion (host side): the reference's loaders over libgcol_io.so.

    load_edge_list      /root/reference/proj/include/gcol/graph_io.hpp:83-106
    save_edge_list      graph_io.hpp:110-117
    load_matrix_market  graph_io.hpp:124-221
    load_graph          /root/reference/proj/tools/gcol_main.cpp:25-35
    read_coloring_file  gcol_main.cpp:72-108

Each returns the canonical CSR (int64 offsets, int32 columns) that
`gcol.Graph` uploads.  Errors carry the reference's classes and messages
(errors.hpp:11-52); the parsing itself is include/gcol_io.hpp (C++)."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgcol_io.so")

FORMAT_AUTO, FORMAT_EDGELIST, FORMAT_MM = 0, 1, 2


class input_error(ValueError):  # errors.hpp:11-14
    pass


class parse_error(RuntimeError):  # errors.hpp:17-28
    def __init__(self, msg: str, line: int):
        super().__init__(msg)
        self.line = line


class unsupported_format_error(RuntimeError):  # errors.hpp:32-35
    pass


class capacity_error(RuntimeError):  # errors.hpp:38-41
    pass


class io_error(RuntimeError):  # errors.hpp:50-53
    pass


_lib: Optional[C.CDLL] = None
_vp = C.c_void_p


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)  # missing library: fail loudly
        L.gcol_io_last_error.restype = C.c_char_p
        L.gcol_io_last_error_line.restype = C.c_uint64
        L.gcol_io_parse.argtypes = [C.c_char_p, C.c_uint64, C.c_int32, C.c_int64, C.POINTER(_vp)]
        L.gcol_io_load.argtypes = [C.c_char_p, C.c_int32, C.POINTER(_vp)]
        L.gcol_io_build_graph.argtypes = [_vp, C.c_uint64, C.c_uint64, C.POINTER(_vp)]
        L.gcol_io_graph_free.argtypes = [_vp]
        L.gcol_io_graph_free.restype = None
        L.gcol_io_num_vertices.argtypes = [_vp]
        L.gcol_io_num_vertices.restype = C.c_int64
        L.gcol_io_num_adjacency.argtypes = [_vp]
        L.gcol_io_num_adjacency.restype = C.c_int64
        L.gcol_io_max_degree.argtypes = [_vp]
        L.gcol_io_max_degree.restype = C.c_int32
        L.gcol_io_offsets.argtypes = [_vp]
        L.gcol_io_offsets.restype = _vp
        L.gcol_io_cols.argtypes = [_vp]
        L.gcol_io_cols.restype = _vp
        L.gcol_io_format_edge_list.argtypes = [_vp, C.POINTER(C.c_char_p)]
        L.gcol_io_format_edge_list.restype = C.c_uint64
        L.gcol_io_save_edge_list.argtypes = [_vp, C.c_char_p]
        L.gcol_io_parse_coloring.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(_vp), C.POINTER(C.c_uint64)]
        L.gcol_io_free.argtypes = [_vp]
        L.gcol_io_free.restype = None
        _lib = L
    return _lib


def _raise(rc: int) -> None:
    L = lib()
    msg = L.gcol_io_last_error().decode()
    if rc == 2:
        raise parse_error(msg, int(L.gcol_io_last_error_line()))
    raise {1: input_error, 3: unsupported_format_error, 4: capacity_error, 5: io_error}.get(rc, RuntimeError)(msg)


def _take(handle) -> Tuple[np.ndarray, np.ndarray]:
    """Copies the handle's CSR into numpy arrays and releases it."""
    L = lib()
    try:
        n, m = L.gcol_io_num_vertices(handle), L.gcol_io_num_adjacency(handle)
        off = np.ctypeslib.as_array(C.cast(L.gcol_io_offsets(handle), C.POINTER(C.c_int64)), (n + 1,)).copy()
        cols = (np.ctypeslib.as_array(C.cast(L.gcol_io_cols(handle), C.POINTER(C.c_int32)), (m,)).copy()
                if m else np.zeros(0, np.int32))
        return off, cols
    finally:
        L.gcol_io_graph_free(handle)


def _parse(text, fmt: int, num_vertices: int) -> Tuple[np.ndarray, np.ndarray]:
    if isinstance(text, str):
        text = text.encode()
    h = _vp()
    rc = lib().gcol_io_parse(text, len(text), fmt, num_vertices, C.byref(h))
    if rc:
        _raise(rc)
    return _take(h)


def load_edge_list(text, num_vertices: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """graph_io.hpp:83-106 on an in-memory source (str or bytes)."""
    return _parse(text, FORMAT_EDGELIST, -1 if num_vertices is None else int(num_vertices))


def load_matrix_market(text) -> Tuple[np.ndarray, np.ndarray]:
    """graph_io.hpp:124-221 on an in-memory source."""
    return _parse(text, FORMAT_MM, -1)


def load_graph(path: str, fmt: str = "auto") -> Tuple[np.ndarray, np.ndarray]:
    """gcol_main.cpp:25-35: by extension unless fmt is 'mm' or 'edgelist'."""
    h = _vp()
    code = {"auto": FORMAT_AUTO, "edgelist": FORMAT_EDGELIST, "mm": FORMAT_MM}[fmt]
    rc = lib().gcol_io_load(os.fsencode(path), code, C.byref(h))
    if rc:
        _raise(rc)
    return _take(h)


def build_graph(pairs, num_vertices: int) -> Tuple[np.ndarray, np.ndarray]:
    """graph.hpp:98-138 over raw (u, v) pairs in any order and orientation."""
    e = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint32).reshape(-1, 2))
    h = _vp()
    rc = lib().gcol_io_build_graph(e.ctypes.data_as(_vp), len(e), int(num_vertices), C.byref(h))
    if rc:
        _raise(rc)
    return _take(h)


def save_edge_list(off: np.ndarray, cols: np.ndarray) -> bytes:
    """graph_io.hpp:110-117: the text load_edge_list reads back."""
    off = np.asarray(off, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int32)
    n = off.size - 1
    out = [f"# {n} vertices, {cols.size // 2} edges\n".encode()]
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    up = cols > rows
    if up.any():
        body = np.stack([rows[up], cols[up].astype(np.int64)], axis=1)
        out.append(("\n".join(f"{a} {b}" for a, b in body.tolist()) + "\n").encode())
    return b"".join(out)


def read_coloring(text) -> np.ndarray:
    """gcol_main.cpp:72-108: one colour per line, -1 = uncoloured."""
    if isinstance(text, str):
        text = text.encode()
    p, k = _vp(), C.c_uint64(0)
    rc = lib().gcol_io_parse_coloring(text, len(text), C.byref(p), C.byref(k))
    if rc:
        _raise(rc)
    try:
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_int32)), (max(1, k.value),))[:k.value].copy()
    finally:
        lib().gcol_io_free(p)

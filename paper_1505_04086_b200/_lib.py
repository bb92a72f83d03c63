"""ctypes binding of libgcol_cuda.so (the C ABI declared in include/gcol_cuda.h).

The library is the product: this module only marshals arguments.  If the
shared object is missing or fails to load, import fails loudly -- there is
no Python/CPU fallback for any coloring operation.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GCOL_CUDA_LIB: another build of the same ABI (A/B tooling); the default is the in-tree library
LIB_PATH = os.environ.get("GCOL_CUDA_LIB") or os.path.join(HERE, "libgcol_cuda.so")

GCOL_OK = 0
GCOL_ERR_INVALID_ARGUMENT = 1
GCOL_ERR_CAPACITY = 2
GCOL_ERR_CUDA = 3
GCOL_ERR_NCCL = 4
GCOL_ERR_ROUND_CAP = 5
GCOL_ERR_VERIFY = 6
GCOL_ERR_NO_DEVICE = 7

GCOL_MEM_HOST = 0
GCOL_MEM_DEVICE = 1

PRIORITY_DEFAULT = 0
PRIORITY_ID_LOW = 1
PRIORITY_ID_HIGH = 2
PRIORITY_DEGREE_ID = 3
PRIORITY_ORDERED = 4

ALG_SEQ = 0
ALG_CATALYUREK = 1
ALG_RSOC = 2


class Options(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("thread_count", C.c_uint32),
        ("chunk_size", C.c_uint64),
        ("min_chunk_size", C.c_uint64),
        ("round_cap", C.c_uint64),
        ("priority", C.c_int32),
        ("k1_blocks_per_sm", C.c_int32),
        ("k1_read_all", C.c_int32),
        ("k1_split_min_degree", C.c_int32),
        ("k1_wide", C.c_int32),
        ("k1_wait_polls", C.c_int32),
        ("reserved", C.c_int32 * 2),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32),
        ("thread_count", C.c_uint32),
        ("rounds", C.c_uint64),
        ("conflicts_total", C.c_uint64),
        ("barrier_events", C.c_uint64),
        ("num_colors", C.c_uint32),
        ("fallback_triggered", C.c_uint32),
        ("wall_time_ns", C.c_uint64),
        ("initial_pass_ns", C.c_uint64),
        ("cpr_len", C.c_uint64),
        ("conflicts_per_round", C.POINTER(C.c_uint64)),
        ("cpr_cap", C.c_uint64),
        ("pairs_logged", C.c_uint64),
        ("round1_candidates", C.c_uint64),
        ("pair_overflow", C.c_uint32),
        ("priority", C.c_int32),
        ("k1_gathers", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("heavy_pass_ns", C.c_uint64),
        ("heavy_rows", C.c_uint64),
    ]


class VerifyReport(C.Structure):
    _fields_ = [
        ("violations", C.c_uint64),
        ("uncolored", C.c_uint64),
        ("conflict_edges", C.c_uint64),
        ("out_of_bound", C.c_uint64),
        ("negative", C.c_uint64),
        ("num_colors", C.c_uint32),
        ("max_color", C.c_int32),
    ]


# Every exported symbol of include/gcol_cuda.h, with its ctypes signature.
_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
SIGNATURES = {
    "gcol_cuda_abi_version": (C.c_int, []),
    "gcol_cuda_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "gcol_cuda_last_error": (C.c_char_p, []),
    "gcol_cuda_graph_create": (C.c_int, [_vp, _vp, _i64, _i64, _i32, _i32, C.POINTER(_vp)]),
    "gcol_cuda_graph_destroy": (C.c_int, [_vp]),
    "gcol_cuda_graph_info": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i32)]),
    "gcol_cuda_color_rsoc": (C.c_int, [_vp, C.POINTER(Options), _vp, _i32, C.POINTER(Stats)]),
    "gcol_cuda_color_rsoc_csr": (C.c_int, [_vp, _vp, _i64, _i64, _i32, C.POINTER(Options), _vp,
                                           C.POINTER(Stats)]),
    "gcol_cuda_color_catalyurek": (C.c_int, [_vp, C.POINTER(Options), _vp, _i32,
                                             C.POINTER(Stats)]),
    "gcol_cuda_run_coloring": (C.c_int, [_vp, _i32, C.POINTER(Options), _vp, _i32,
                                         C.POINTER(Stats)]),
    "gcol_cuda_first_fit_sequential": (C.c_int, [_vp, _vp, _i32]),
    "gcol_cuda_tentative_snapshot": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _i32]),
    "gcol_cuda_detect_conflicts": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, _i32]),
    "gcol_cuda_detect_and_recolor": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp, C.POINTER(_i64),
                                               _i32]),
    "gcol_cuda_verify_coloring": (C.c_int, [_vp, _vp, _i64, _i32, C.POINTER(VerifyReport), _vp,
                                            _vp, _vp, _i64]),
    "gcol_cuda_count_colors": (C.c_int, [_vp, _vp, _i64, _i32, C.POINTER(C.c_uint32)]),
    "gcol_cuda_ipc_export": (C.c_int, [_vp, _vp, C.POINTER(C.c_uint64)]),
    "gcol_cuda_ipc_import": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_void_p)]),
    "gcol_cuda_ipc_close": (C.c_int, [_vp, C.c_uint64]),
    "gcol_cuda_partition_set": (C.c_int, [_vp, _i32, _i32, _vp]),
    "gcol_cuda_k1_owned": (C.c_int, [_vp, C.POINTER(Options), _vp, C.POINTER(Stats)]),
    "gcol_cuda_candidates": (C.c_int, [_vp, _i32, _vp, _vp, C.POINTER(C.c_int64)]),
    "gcol_cuda_k1_range": (C.c_int, [_vp, C.POINTER(Options), _vp, _i64, _i64, C.POINTER(Stats)]),
    "gcol_cuda_detect_range": (C.c_int, [_vp, _i32, _vp, _i64, _i64, _vp, C.POINTER(_i64)]),
    "gcol_cuda_round_list": (C.c_int, [_vp, _i32, _vp, _vp, _i64, _vp, C.POINTER(_i64)]),
    "gcol_cuda_scatter_colors": (C.c_int, [_vp, _vp, _vp, _vp, _i64]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python paper_1505_04086_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()


def last_error() -> str:
    msg = LIB.gcol_cuda_last_error()
    return msg.decode() if msg else ""

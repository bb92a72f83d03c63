"""B200-native (sm_100a) RSOC optimistic graph coloring (arXiv 1505.04086).

The coloring path is libgcol_cuda.so (hand-written CUDA kernels behind the C
ABI in include/gcol_cuda.h); `gcol` mirrors the reference's C++ interface.

The library is loaded on first use of a coloring name (PEP 562 lazy
attributes), not by `import paper_1505_04086_b200`: workload generation
(`graphs`) must not map libgcol_cuda.so, so that bench.py's reference arm
runs the reference with none of this package's native code in the process.
Loading still fails loudly when the library is absent (no CPU fallback).
"""
import importlib

_GCOL_NAMES = ("Algorithm", "ColoringRun", "ColoringStats", "ConflictReport", "Graph",
               "ParallelOptions", "Priority", "build_graph", "capacity_error", "color_rsoc",
               "count_colors", "detect_conflicts", "first_fit_sequential", "input_error",
               "run_coloring", "verification_error", "verify_coloring")

__all__ = list(_GCOL_NAMES)


def __getattr__(name):
    if name in _GCOL_NAMES:
        return getattr(importlib.import_module(".gcol", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

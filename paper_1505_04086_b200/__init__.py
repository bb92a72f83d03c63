"""B200-native (sm_100a) RSOC optimistic graph coloring (arXiv 1505.04086).

The coloring path is libgcol_cuda.so (hand-written CUDA kernels behind the C
ABI in include/gcol_cuda.h); `gcol` mirrors the reference's C++ interface.
"""
from . import gcol  # noqa: F401  (loads libgcol_cuda.so; fails loudly if absent)
from .gcol import (Algorithm, ColoringRun, ColoringStats, ConflictReport, Graph,  # noqa: F401
                   ParallelOptions, Priority, build_graph, capacity_error, color_rsoc,
                   count_colors, detect_conflicts, first_fit_sequential, input_error,
                   run_coloring, verification_error, verify_coloring)

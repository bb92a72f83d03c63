"""Build recipe for libgcol_cuda.so (sm_100a) -- in-tree, no JIT cache.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared, cudart
linked statically so the library carries no dependency on a torch-bundled
runtime.  The .so lands next to this file and travels with the repo
snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgcol_cuda.so")
SOURCES = ["gcol_cuda.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xcompiler", "-pthread",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
    "-cudart", "static",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in os.listdir(CSRC) if d.endswith((".cu", ".cuh", ".h"))]
    deps += [os.path.join(REPO, "include", "gcol_cuda.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    extra = os.environ.get("GCOL_NVCC_EXTRA", "").split()  # experiments, e.g. -DGCOL_DEBUG_HEAVY
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-shared", "-I", CSRC, "-I", os.path.join(REPO, "include"),
           "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed building libgcol_cuda.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


IO_LIB = os.path.join(HERE, "libgcol_io.so")
CLI_BIN = os.path.join(HERE, "gcol_b200")


def _newer(target: str, deps) -> bool:
    return os.path.exists(target) and all(os.path.getmtime(target) > os.path.getmtime(d) for d in deps)


def build_io() -> str:
    """libgcol_io.so: the host-side text loaders behind include/gcol_io.h (g++ only)."""
    deps = [os.path.join(CSRC, "gcol_io_abi.cpp"), os.path.join(REPO, "include", "gcol_io.hpp"),
            os.path.join(REPO, "include", "gcol_io.h")]
    if _newer(IO_LIB, deps):
        return IO_LIB
    cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-I", os.path.join(REPO, "include"),
           "-o", IO_LIB, deps[0]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("building libgcol_io.so failed")
    return IO_LIB


def build_cli() -> str:
    """gcol_b200: the color / verify / bench front-end over the C ABI."""
    lib = build()
    src = os.path.join(REPO, "tools", "gcol_b200_cli.cpp")
    deps = [src, lib, os.path.join(REPO, "include", "gcol_io.hpp"), os.path.join(REPO, "include", "gcol_cuda.h")]
    if _newer(CLI_BIN, deps):
        return CLI_BIN
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(REPO, "include"), src, "-o", CLI_BIN,
           "-L", HERE, "-lgcol_cuda", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("building gcol_b200 failed")
    return CLI_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_io())
    print(build_cli())


ADAPTER_SRC = os.path.join(REPO, "tests", "cpp", "adapter_check.cpp")
ADAPTER_BIN = os.path.join(REPO, "tests", "cpp", "adapter_check")
REF_INCLUDE = os.environ.get("GCOL_REF_INCLUDE", "/root/reference/proj/include")


def build_adapter_check() -> str | None:
    """C++ program using the reference's own headers + include/gcol_cuda.hpp
    against libgcol_cuda.so (only where the reference headers exist; the
    binary travels to the GPU box)."""
    if not os.path.isdir(os.path.join(REF_INCLUDE, "gcol")):
        return None
    lib = build()
    if os.path.exists(ADAPTER_BIN) and os.path.getmtime(ADAPTER_BIN) > max(
            os.path.getmtime(lib), os.path.getmtime(ADAPTER_SRC),
            os.path.getmtime(os.path.join(REPO, "include", "gcol_cuda.hpp"))):
        return ADAPTER_BIN
    cmd = ["g++", "-std=c++20", "-O2", "-I", REF_INCLUDE, "-I", os.path.join(REPO, "include"),
           ADAPTER_SRC, "-o", ADAPTER_BIN, "-L", HERE, "-lgcol_cuda",
           "-Wl,-rpath,$ORIGIN/../../paper_1505_04086_b200"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("building tests/cpp/adapter_check failed")
    return ADAPTER_BIN

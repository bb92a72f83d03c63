"""Generates tests/golden/*.npz from THE REFERENCE ITSELF.

Run in the build container (needs oracle/_ref/libgcolref.so, i.e. the
reference's header-only gcol library compiled from /root/reference by
oracle/Makefile).  The GPU box never runs this; it only reads the fixtures.

Fixtures pin:
  - build_graph          (graph.hpp:98-138)      canonical CSR per edge list
  - first_fit_sequential (coloring.hpp:110-116)  colours
  - smallest_available_color (coloring.hpp:95-106) over random snapshots
  - detect_conflicts     (coloring.hpp:133-141)  full and partial worklists
  - verify_coloring      (coloring.hpp:159-177)  violation lists
  - count_colors         (coloring.hpp:181-196)
  - color_rsoc @ 1 thread (parallel.hpp:253-319) colours + stats
  - lockstep_color       (lockstep.hpp:37-78)    traces
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle  # noqa: E402


def kat_graphs():
    g = {}
    g["path3"] = ([(0, 1), (1, 2)], 3)
    g["k3"] = ([(0, 1), (1, 2), (0, 2)], 3)
    g["c5"] = ([(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)], 5)
    g["empty"] = ([], 0)
    g["lone"] = ([], 1)
    g["pair"] = ([(0, 1)], 2)
    g["dup_loop"] = ([(0, 1), (1, 0), (1, 1)], 2)
    g["k12"] = ([(u, v) for u in range(12) for v in range(u + 1, 12)], 12)
    g["star200"] = ([(0, v) for v in range(1, 200)], 200)
    g["star_gap"] = ([(0, 1), (0, 2)], 3)
    return g


def random_edges(rng, n, avg):
    m = int(n * avg / 2)
    if n < 2:
        return np.zeros((0, 2), np.uint32)
    return rng.integers(0, n, size=(m, 2), dtype=np.int64).astype(np.uint32)


def heavy_graph(rng):
    """A graph with rows in every width class: small, warp (64..1023), CTA
    (>1023) and a hub above the 16384-colour block window."""
    n = 40000
    e = [random_edges(rng, n, 6.0)]
    hub = 7
    e.append(np.stack([np.full(20000, hub), rng.choice(n, 20000, replace=False)], 1))
    for h, d in ((100, 1500), (200, 700), (300, 64), (400, 63), (500, 1024), (600, 1023)):
        e.append(np.stack([np.full(d, h), rng.choice(n, d, replace=False)], 1))
    return np.concatenate(e).astype(np.uint32), n


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref/libgcolref.so missing: run `make -C oracle` first")
    rng = np.random.default_rng(20150515)
    cases = []
    for name, (edges, n) in kat_graphs().items():
        cases.append((name, np.asarray(edges, dtype=np.uint32).reshape(-1, 2), n))
    for i in range(60):
        n = int(rng.integers(1, 400))
        avg = float(rng.uniform(0.5, 9.0))
        cases.append((f"rand{i}", random_edges(rng, n, avg), n))
    for i in range(4):
        n = int(rng.integers(1500, 3000))
        cases.append((f"mid{i}", random_edges(rng, n, float(rng.uniform(8, 24))), n))
    he, hn = heavy_graph(rng)
    cases.append(("heavy", he, hn))

    out = {}
    names = []
    for name, edges, n in cases:
        names.append(name)
        R = oracle.RefGraph.from_edges(edges, n)
        csr = R.csr()
        if not (name.startswith("mid") or name == "heavy"):
            out[f"{name}/edges"] = edges  # build_graph pin; larger graphs keep only the CSR
        out[f"{name}/n"] = np.array([n], np.int64)
        out[f"{name}/off"] = csr.off.astype(np.int64)
        out[f"{name}/cols"] = csr.cols.astype(np.int32)
        out[f"{name}/ff"] = R.first_fit_sequential()
        deg = np.diff(csr.off.astype(np.int64))
        # random narrow-palette colouring with holes (test_coloring.cpp:124-141)
        pal = rng.integers(-1, 3, size=n).astype(np.int32)
        out[f"{name}/pal"] = pal
        allv = np.arange(n, dtype=np.uint32)
        out[f"{name}/detect_all"] = np.array(R.detect_conflicts(pal, allv), np.int32)
        out[f"{name}/detect_even"] = np.array(R.detect_conflicts(pal, allv[::2]), np.int32)
        viol = R.verify_coloring(pal)
        out[f"{name}/verify"] = np.array(viol, np.int64).reshape(-1, 3)
        # snapshot colouring spanning colours above the degree bound
        snap = np.where(rng.random(n) < 0.2, -1,
                        rng.integers(0, np.maximum(deg, 1) + 3)).astype(np.int32) if n else \
            np.zeros(0, np.int32)
        if name == "heavy":  # hub neighbours carry 18000 distinct colours
            hub_nb = csr.cols[csr.off[7]:csr.off[8]].astype(np.int64)
            snap[hub_nb[:18000]] = np.arange(18000, dtype=np.int32)
        out[f"{name}/snap"] = snap
        out[f"{name}/snap_sac"] = np.array([R.smallest_available_color(snap, v) for v in range(n)],
                                           np.int32)
        colors, st = R.color("rsoc", 1)
        out[f"{name}/rsoc1"] = colors
        out[f"{name}/rsoc1_stats"] = np.array([st["rounds"], st["conflicts_total"],
                                               st["barrier_events"], st["num_colors"]], np.int64)
        try:
            out[f"{name}/count_ff"] = np.array([oracle.ref_count_colors(out[f"{name}/ff"])], np.int64)
        except Exception:
            out[f"{name}/count_ff"] = np.array([-1], np.int64)
    # lockstep traces (test_lockstep.cpp)
    lock = {}
    for lname, edges, n, lanes, cap in (
            ("pair_split", [(0, 1)], 2, [0, 1], 10),
            ("pair_one", [(0, 1)], 2, [0, 0], 10),
            ("tri_one", [(0, 1), (1, 2), (0, 2)], 3, [0, 0, 0], 10),
            ("iso", [], 3, [0, 1, 2], 5)):
        R = oracle.RefGraph.from_edges(np.asarray(edges, np.uint32).reshape(-1, 2), n)
        conv, rounds, trace = R.lockstep_color(lanes, cap)
        lock[f"{lname}/edges"] = np.asarray(edges, np.uint32).reshape(-1, 2)
        lock[f"{lname}/n"] = np.array([n], np.int64)
        lock[f"{lname}/lanes"] = np.asarray(lanes, np.uint32)
        lock[f"{lname}/cap"] = np.array([cap], np.int64)
        lock[f"{lname}/result"] = np.array([int(conv), rounds], np.int64)
        lock[f"{lname}/trace"] = np.asarray(trace, np.int32)
    np.savez_compressed(os.path.join(HERE, "ref_coloring.npz"), names=np.array(names), **out)
    np.savez_compressed(os.path.join(HERE, "ref_lockstep.npz"), **lock)
    print(f"wrote {len(names)} graphs")


if __name__ == "__main__":
    main()

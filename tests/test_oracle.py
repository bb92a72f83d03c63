"""CPU: pin the oracle (oracle/gcol_oracle.c) before trusting it.

(1) the known-answer tests of the reference's own suite
    (proj/tests/test_coloring.cpp, test_parallel.cpp, test_lockstep.cpp),
(2) the golden fixtures generated from the reference itself
    (tests/golden/make_golden.py), and
(3) the reference library (oracle/_ref) run side by side, when built here.
"""
import numpy as np
import pytest

from tests.golden_util import coloring_fixtures, lockstep_fixtures


def csr_of(oracle_mod, case):
    return oracle_mod.CSR(case["off"], case["cols"])


# --- (1) reference KATs ------------------------------------------------------------
def test_smallest_available_color_kats(oracle_mod):  # test_coloring.cpp:30-49
    o = oracle_mod
    tri = o.build_graph([(0, 1), (1, 2), (0, 2)], 3)
    assert o.smallest_available_color(tri, [-1, -1, -1], 0) == 0
    assert o.smallest_available_color(tri, [0, -1, 1], 1) == 2
    star = o.build_graph([(0, 1), (0, 2)], 3)
    assert o.smallest_available_color(star, [-1, 0, 2], 0) == 1


def test_first_fit_frozen_cases(oracle_mod):  # test_coloring.cpp:64-78
    o = oracle_mod
    assert list(o.first_fit_sequential(o.build_graph([(0, 1), (1, 2)], 3))) == [0, 1, 0]
    assert list(o.first_fit_sequential(o.build_graph([(0, 1), (1, 2), (0, 2)], 3))) == [0, 1, 2]
    c5 = o.build_graph([(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)], 5)
    assert list(o.first_fit_sequential(c5)) == [0, 1, 0, 1, 2]
    assert o.first_fit_sequential(o.build_graph([], 0)).size == 0


def test_detect_kats(oracle_mod):  # test_coloring.cpp:108-122
    o = oracle_mod
    pair = o.build_graph([(0, 1)], 2)
    assert o.detect_conflicts(pair, [0, 0], [0, 1]) == [0]
    tri = o.build_graph([(0, 1), (1, 2), (0, 2)], 3)
    assert o.detect_conflicts(tri, [0, 0, 0], [0, 1, 2]) == [0, 1]
    assert o.detect_conflicts(tri, o.first_fit_sequential(tri), [0, 1, 2]) == []


def test_verify_kats(oracle_mod):  # test_coloring.cpp:143-163
    o = oracle_mod
    path = o.build_graph([(0, 1), (1, 2)], 3)
    assert o.verify_coloring(path, [0, 1, 0]) == []
    assert o.verify_coloring(path, [0, 0, 1]) == [(0, 1, 0)]
    assert o.verify_coloring(path, [0, 1, -1]) == [(2, 0xFFFFFFFF, -1)]


def test_count_colors_kats(oracle_mod):  # test_coloring.cpp:165-181
    o = oracle_mod
    assert o.count_colors([0, 1, 0]) == 2
    assert o.count_colors([0, 1, 2]) == 3
    assert o.count_colors([0, 0, 0]) == 1
    assert o.count_colors([]) == 0
    assert o.count_colors([0, -1]) == -1   # incomplete -> input_error
    assert o.count_colors([-5]) == -2      # negative -> input_error
    assert o.count_colors([0, 5]) == 2     # distinct, not 1 + max


def check_run(g, colors, st, threads, algorithm):
    """test_parallel.cpp:18-36 invariants."""
    o_ok = all(c >= 0 for c in colors)
    assert o_ok
    assert st["thread_count"] == threads
    assert st["rounds"] >= 1
    assert len(st["conflicts_per_round"]) == st["rounds"]
    assert st["conflicts_total"] == sum(st["conflicts_per_round"])
    if not st["fallback_triggered"]:
        assert st["conflicts_per_round"][-1] == 0
    if algorithm == "rsoc":
        assert st["barrier_events"] == st["rounds"] + 1
    else:
        assert st["barrier_events"] == 2 * st["rounds"]
    assert st["num_colors"] <= g.max_degree + 1


def test_parallel_oracle_invariants(oracle_mod):  # test_parallel.cpp:40-116
    o = oracle_mod
    rng = np.random.default_rng(707)
    for _ in range(6):
        n = int(rng.integers(50, 2000))
        e = rng.integers(0, n, size=(n * 4, 2))
        g = o.build_graph(e, n)
        seq = o.first_fit_sequential(g)
        for t in (1, 2, 4, 8):
            for alg in ("rsoc", "catalyurek"):
                colors, st = o.color_parallel(g, t, alg)
                check_run(g, colors, st, t, alg)
                assert o.verify_coloring(g, colors) == []
                assert st["num_colors"] == o.count_colors(colors)
                if t == 1:  # single-thread equivalence (acceptance criterion 3)
                    assert np.array_equal(colors, seq)
                    assert st["rounds"] == 1 and st["conflicts_total"] == 0
    k12 = o.build_graph([(u, v) for u in range(12) for v in range(u + 1, 12)], 12)
    star = o.build_graph([(0, v) for v in range(1, 200)], 200)
    for t in (1, 2, 4, 8):
        assert o.color_parallel(k12, t, "rsoc")[1]["num_colors"] == 12
        assert o.color_parallel(star, t, "catalyurek")[1]["num_colors"] == 2
    empty = o.build_graph([], 0)
    _, st = o.color_parallel(empty, 4, "rsoc")
    assert st["rounds"] == 1 and st["conflicts_per_round"] == [0] and st["barrier_events"] == 2
    with pytest.raises(ValueError):
        o.color_parallel(k12, 0, "rsoc")


def test_lockstep_kats(oracle_mod):  # test_lockstep.cpp:14-58
    o = oracle_mod
    pair = o.build_graph([(0, 1)], 2)
    conv, rounds, trace = o.lockstep_color(pair, [0, 1], 10)
    assert not conv and rounds == 10
    for r in range(10):
        e = 0 if r % 2 == 0 else 1
        assert list(trace[r]) == [e, e]
    conv, rounds, trace = o.lockstep_color(pair, [0, 0], 10)
    assert conv and rounds == 1 and list(trace[0]) == [0, 1]
    iso = o.build_graph([], 3)
    conv, rounds, trace = o.lockstep_color(iso, [0, 1, 2], 5)
    assert conv and rounds == 1 and list(trace[-1]) == [0, 0, 0]
    conv, rounds, _ = o.lockstep_color(o.build_graph([], 0), [], 5)
    assert conv and rounds == 0


# --- (2) golden fixtures from the reference ----------------------------------------
@pytest.mark.parametrize("name", list(coloring_fixtures().keys()))
def test_oracle_matches_reference_golden(oracle_mod, name):
    o = oracle_mod
    case = coloring_fixtures()[name]
    n = int(case["n"][0])
    if "edges" in case:  # build_graph pin
        g = o.build_graph(case["edges"], n)
        assert np.array_equal(g.off.astype(np.int64), case["off"])
        assert np.array_equal(g.cols.astype(np.int32), case["cols"])
    g = csr_of(o, case)
    assert np.array_equal(o.first_fit_sequential(g), case["ff"])
    allv = np.arange(n)
    assert o.detect_conflicts(g, case["pal"], allv) == list(case["detect_all"])
    assert o.detect_conflicts(g, case["pal"], allv[::2]) == list(case["detect_even"])
    assert o.verify_coloring(g, case["pal"]) == [tuple(int(x) for x in r) for r in case["verify"]]
    assert np.array_equal(o.tentative_snapshot(g, case["snap"]), case["snap_sac"])
    colors, st = o.color_parallel(g, 1, "rsoc")
    assert np.array_equal(colors, case["rsoc1"])
    assert [st["rounds"], st["conflicts_total"], st["barrier_events"], st["num_colors"]] == \
        list(case["rsoc1_stats"])
    assert o.count_colors(case["ff"]) == int(case["count_ff"][0])


def test_oracle_lockstep_golden(oracle_mod):
    o = oracle_mod
    for name, case in lockstep_fixtures().items():
        g = o.build_graph(case["edges"], int(case["n"][0]))
        conv, rounds, trace = o.lockstep_color(g, case["lanes"], int(case["cap"][0]))
        assert [int(conv), rounds] == list(case["result"]), name
        assert np.array_equal(np.asarray(trace).reshape(case["trace"].shape), case["trace"]), name


# --- (3) the reference library side by side ------------------------------------------
def test_oracle_vs_reference_library_multithreaded(oracle_mod):
    o = oracle_mod
    if not o.ref_available():
        pytest.skip("oracle/_ref not built on this machine")
    rng = np.random.default_rng(4242)
    for _ in range(5):
        n = int(rng.integers(100, 3000))
        e = rng.integers(0, n, size=(int(n * rng.uniform(2, 10)), 2))
        R = o.RefGraph.from_edges(e, n)
        g = R.csr()
        seq = o.first_fit_sequential(g)
        assert np.array_equal(seq, R.first_fit_sequential())
        for t in (2, 4, 8):
            rc, rst = R.color("rsoc", t)
            oc, ost = o.color_parallel(g, t, "rsoc")
            # schedules differ run to run; the invariants and the palette band must hold
            check_run(g, rc, rst, t, "rsoc")
            check_run(g, oc, ost, t, "rsoc")
            assert abs(ost["num_colors"] - rst["num_colors"]) <= max(2, rst["num_colors"] // 10)

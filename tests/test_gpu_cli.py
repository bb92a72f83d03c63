"""gcol_b200 on the GPU: the color / verify / bench cases of the reference's
CLI integration test (/root/reference/proj/tests/test_cli.cpp:110-225), run
against the binary built over the C ABI."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle
from paper_1505_04086_b200 import graph_io

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_1505_04086_b200", "gcol_b200")


def run_cli(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([CLI, *args], capture_output=True, text=True, env=e, timeout=300)
    return r.returncode, r.stdout + r.stderr


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    (d / "path.el").write_text("0 1\n1 2\n")
    (d / "tri.mtx").write_text("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n2 1\n3 1\n3 2\n")
    rng = np.random.default_rng(3)
    pairs = rng.integers(0, 3000, size=(24000, 2))
    (d / "er.el").write_text("".join(f"{u} {v}\n" for u, v in pairs.tolist()))
    return d


def test_cli_color(files):
    d = files
    rc, out = run_cli("color", str(d / "path.el"), "--algorithm", "seq")
    assert rc == 0, out
    st = json.loads(out)
    assert st["algorithm"] == "seq" and st["num_colors"] == 2 and st["rounds"] == 1
    assert st["graph_stats"] == {"max_degree": 2, "num_edges": 2, "num_vertices": 3}
    assert '"algorithm": "seq"' in out and '"num_colors": 2' in out  # dump(2) spelling
    rc, out = run_cli("color", str(d / "path.el"), "--algorithm", "rsoc", "--threads", "3",
                      "--output", str(d / "stats.json"), "--coloring-output", str(d / "colors.txt"))
    assert rc == 0, out
    assert "colored 3 vertices with 2 colors" in out
    st = json.loads((d / "stats.json").read_text())
    assert st["barrier_events"] == st["rounds"] + 1 and st["thread_count"] == 3
    assert st["conflicts_per_round"][-1] == 0 and st["fallback_triggered"] is False
    assert (d / "colors.txt").read_text() == "0\n1\n0\n"
    assert run_cli("color", str(d / "path.el"), "--algorithm", "catalyurek", "--threads", "2",
                   env={"GCOL_CHUNK_SIZE": "16"})[0] == 0
    rc, out = run_cli("color", str(d / "tri.mtx"), "--algorithm", "rsoc", "--threads", "4")
    assert rc == 0 and '"num_colors": 3' in out
    assert run_cli("color", str(d / "tri.mtx"), "--format", "mm")[0] == 0


def test_cli_color_checked_by_the_oracle(files):
    d = files
    for alg in ("seq", "catalyurek", "rsoc"):
        rc, out = run_cli("color", str(d / "er.el"), "--algorithm", alg, "--coloring-output", str(d / f"{alg}.col"))
        assert rc == 0, out
        c = graph_io.read_coloring((d / f"{alg}.col").read_text())
        off, cols = graph_io.load_graph(str(d / "er.el"))
        g = oracle.CSR(off, cols)
        assert oracle.verify_coloring(g, c) == []
        assert json.loads(out)["num_colors"] == oracle.count_colors(c)
        if alg == "seq":
            assert np.array_equal(c, oracle.first_fit_sequential(g))


def test_cli_verify(files):
    d = files
    (d / "good.col").write_text("0\n1\n0\n")
    (d / "bad.col").write_text("0\n0\n1\n")
    (d / "hole.col").write_text("0\n-1\n0\n")
    rc, out = run_cli("verify", str(d / "path.el"), "--coloring", str(d / "good.col"))
    assert rc == 0 and "proper coloring with 2 colors" in out
    rc, out = run_cli("verify", str(d / "path.el"), "--coloring", str(d / "bad.col"))
    assert rc == 3 and "edge (0, 1): both endpoints have color 0" in out and "1 violation(s)" in out
    rc, out = run_cli("verify", str(d / "path.el"), "--coloring", str(d / "hole.col"))
    assert rc == 3 and "vertex 1 is uncolored" in out


def test_cli_bench(files):
    d = files
    rc, out = run_cli("bench", str(d / "er.el"), "--algorithms", "seq,rsoc", "--threads", "1,2", "--repeats", "2",
                      "--output", str(d / "rep.json"), "--csv", str(d / "runs.csv"))
    assert rc == 0, out
    assert "speedup of rsoc over seq at 1 thread(s)" in out and "graph er.el: 3000 vertices" in out
    csv = (d / "runs.csv").read_text()
    assert csv.startswith("algorithm,threads,run_index,rounds,conflicts_total,num_colors,wall_time_ns\n")
    assert csv.count("\n") == 9  # header + 2 algorithms * 2 thread counts * 2 repeats
    rep = json.loads((d / "rep-rsoc.json").read_text())
    assert rep["algorithm"] == "rsoc" and rep["graph_name"] == "er.el" and rep["repeats"] == 2
    assert rep["thread_counts"] == [1, 2] and len(rep["runs"]) == 4 and len(rep["aggregate"]) == 2
    a = rep["aggregate"][0]
    runs = rep["runs"][:2]
    assert a["wall_time_ns_min"] == min(r["wall_time_ns"] for r in runs)
    assert a["wall_time_ns_max"] == max(r["wall_time_ns"] for r in runs)
    assert a["num_colors_median"] == sorted(r["num_colors"] for r in runs)[0]  # lower median
    assert abs(a["wall_time_ns_mean"] - sum(r["wall_time_ns"] for r in runs) / 2) < 1
    assert json.loads((d / "rep-seq.json").read_text())["algorithm"] == "seq"
    rc, out = run_cli("bench", str(d / "er.el"), "--algorithms", "catalyurek", "--threads", "1", "--repeats", "2",
                      "--output", str(d / "single.json"))
    assert rc == 0 and (d / "single.json").exists()
    assert run_cli("bench", str(d / "er.el"), "--algorithms", "magic")[0] == 2
    assert run_cli("bench", str(d / "er.el"), "--threads", "0")[0] == 2

"""CPU: reports in the reference's schema (bench.hpp:62-227)."""
import io
import json

from paper_1505_04086_b200 import gcol, report


def _fake_report():
    runs = []
    for tc in (1, 4):
        for r in range(3):
            runs.append(gcol.ColoringStats(algorithm=gcol.Algorithm.rsoc, thread_count=tc,
                                           rounds=2 + r, conflicts_total=10 * r,
                                           conflicts_per_round=[10 * r, 0][:2],
                                           barrier_events=3 + r, num_colors=7 + r,
                                           wall_time_ns=1000 * (r + 1)))
    rep = report.BenchReport("tri", gcol.Algorithm.rsoc,
                             {"num_vertices": 9, "num_edges": 16, "max_degree": 6}, 3, [1, 4],
                             runs)
    rep.aggregate = [report._aggregate(1, runs[:3]), report._aggregate(4, runs[3:])]
    return rep


def test_json_schema_matches_bench_hpp():
    j = to = report.to_json(_fake_report())
    json.dumps(j)
    # bench.hpp:194-203
    assert list(j) == ["graph_name", "algorithm", "graph_stats", "repeats", "thread_counts",
                       "runs", "aggregate"]
    assert list(j["graph_stats"]) == ["num_vertices", "num_edges", "max_degree"]
    # bench.hpp:164-176
    assert list(j["runs"][0]) == ["algorithm", "thread_count", "rounds", "conflicts_total",
                                  "conflicts_per_round", "barrier_events", "num_colors",
                                  "wall_time_ns", "fallback_triggered"]
    # bench.hpp:184-192
    assert list(j["aggregate"][0]) == ["thread_count", "wall_time_ns_mean", "wall_time_ns_min",
                                       "wall_time_ns_max", "conflicts_total_mean",
                                       "rounds_mean", "num_colors_median"]
    a = to["aggregate"][0]
    assert a["wall_time_ns_mean"] == 2000 and a["wall_time_ns_min"] == 1000
    assert a["num_colors_median"] == 8 and a["rounds_mean"] == 3
    assert j["algorithm"] == "rsoc"


def test_csv_rows_and_header():
    text = report.csv_string(_fake_report())
    lines = text.strip().split("\n")
    assert lines[0] == "algorithm,threads,run_index,rounds,conflicts_total,num_colors,wall_time_ns"
    assert lines[1] == "rsoc,1,0,2,0,7,1000"
    assert lines[4] == "rsoc,4,0,2,0,7,1000"
    assert len(lines) == 7


def test_relative_speedup():
    a, b = _fake_report(), _fake_report()
    for s in b.runs:
        s.wall_time_ns *= 3
    b.aggregate = [report._aggregate(1, b.runs[:3]), report._aggregate(4, b.runs[3:])]
    assert report.relative_speedup(a, b) == [(1, 3.0), (4, 3.0)]

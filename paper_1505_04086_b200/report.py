"""Benchmark reports in the reference's schema (bench.hpp:62-227), over the
device algorithms, so B200 runs diff against the reference's own reports.

    rep = run_benchmark(g, "tri", gcol.Algorithm.rsoc, [1, 16], repeats=10)
    json.dumps(to_json(rep));  write_csv(sys.stdout, rep)

`thread_counts` are recorded like the reference records them; on the device
they change nothing (the ABI's `thread_count` is bookkeeping only)."""
from __future__ import annotations

import io
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, TextIO, Tuple

from . import gcol

CSV_HEADER = "algorithm,threads,run_index,rounds,conflicts_total,num_colors,wall_time_ns"


@dataclass
class ThreadAggregate:  # bench.hpp:63-71
    thread_count: int = 1
    wall_time_ns_mean: float = 0.0
    wall_time_ns_min: int = 0
    wall_time_ns_max: int = 0
    conflicts_total_mean: float = 0.0
    rounds_mean: float = 0.0
    num_colors_median: int = 0


@dataclass
class BenchReport:  # bench.hpp:75-83
    graph_name: str
    algorithm: gcol.Algorithm
    graph_stats: Dict[str, int]
    repeats: int
    thread_counts: List[int]
    runs: List[gcol.ColoringStats] = field(default_factory=list)
    aggregate: List[ThreadAggregate] = field(default_factory=list)


def _aggregate(tc: int, runs: Sequence[gcol.ColoringStats]) -> ThreadAggregate:
    """bench.hpp:87-110 (lower median of the colour counts)."""
    colors = sorted(s.num_colors for s in runs)
    k = len(runs)
    return ThreadAggregate(
        thread_count=tc,
        wall_time_ns_mean=sum(s.wall_time_ns for s in runs) / k,
        wall_time_ns_min=min(s.wall_time_ns for s in runs),
        wall_time_ns_max=max(s.wall_time_ns for s in runs),
        conflicts_total_mean=sum(s.conflicts_total for s in runs) / k,
        rounds_mean=sum(s.rounds for s in runs) / k,
        num_colors_median=colors[(len(colors) - 1) // 2])


def run_benchmark(g: gcol.Graph, graph_name: str, algorithm: gcol.Algorithm,
                  thread_counts: Sequence[int], repeats: int,
                  opt: Optional[gcol.ParallelOptions] = None, colors_out=None) -> BenchReport:
    """bench.hpp:115-150: `repeats` verified runs per thread count.  A run
    that is not proper and complete raises verification_error (the device
    verifies every run; the reference re-verifies on the host)."""
    if repeats < 1:
        raise gcol.input_error("run_benchmark: repeats must be at least 1")
    if not thread_counts:
        raise gcol.input_error("run_benchmark: need at least one thread count")
    if any(tc < 1 for tc in thread_counts):
        raise gcol.input_error("run_benchmark: thread counts must be at least 1")
    rep = BenchReport(graph_name=graph_name, algorithm=gcol.Algorithm(algorithm),
                      graph_stats={"num_vertices": g.num_vertices(),
                                   "num_edges": g.num_edges(),
                                   "max_degree": g.max_degree()},
                      repeats=repeats, thread_counts=list(thread_counts))
    for tc in thread_counts:
        begin = len(rep.runs)
        for _ in range(repeats):
            run = gcol.run_coloring(g, algorithm, tc, opt, colors_out=colors_out)
            rep.runs.append(run.stats)
        rep.aggregate.append(_aggregate(tc, rep.runs[begin:]))
    return rep


def relative_speedup(a: BenchReport, b: BenchReport) -> List[Tuple[int, float]]:
    """bench.hpp:153-162: mean wall time of b / mean wall time of a per
    shared thread count (> 1: a is faster)."""
    out = []
    for ta in a.aggregate:
        for tb in b.aggregate:
            if ta.thread_count == tb.thread_count and ta.wall_time_ns_mean > 0:
                out.append((ta.thread_count, tb.wall_time_ns_mean / ta.wall_time_ns_mean))
    return out


def stats_to_json(s: gcol.ColoringStats) -> Dict:
    """bench.hpp:164-176."""
    return {"algorithm": gcol.to_string(s.algorithm), "thread_count": s.thread_count,
            "rounds": s.rounds, "conflicts_total": s.conflicts_total,
            "conflicts_per_round": list(s.conflicts_per_round),
            "barrier_events": s.barrier_events, "num_colors": s.num_colors,
            "wall_time_ns": s.wall_time_ns, "fallback_triggered": bool(s.fallback_triggered)}


def to_json(rep: BenchReport) -> Dict:
    """bench.hpp:178-204."""
    return {
        "graph_name": rep.graph_name,
        "algorithm": gcol.to_string(rep.algorithm),
        "graph_stats": dict(rep.graph_stats),
        "repeats": rep.repeats,
        "thread_counts": list(rep.thread_counts),
        "runs": [stats_to_json(s) for s in rep.runs],
        "aggregate": [{"thread_count": a.thread_count,
                       "wall_time_ns_mean": a.wall_time_ns_mean,
                       "wall_time_ns_min": a.wall_time_ns_min,
                       "wall_time_ns_max": a.wall_time_ns_max,
                       "conflicts_total_mean": a.conflicts_total_mean,
                       "rounds_mean": a.rounds_mean,
                       "num_colors_median": a.num_colors_median} for a in rep.aggregate],
    }


def write_csv_rows(out: TextIO, rep: BenchReport) -> None:
    """bench.hpp:210-221: one row per run, run_index within a thread count."""
    i = 0
    for tc in rep.thread_counts:
        for r in range(rep.repeats):
            s = rep.runs[i]
            out.write(f"{gcol.to_string(s.algorithm)},{tc},{r},{s.rounds},{s.conflicts_total},"
                      f"{s.num_colors},{s.wall_time_ns}\n")
            i += 1


def write_csv(out: TextIO, rep: BenchReport) -> None:
    """bench.hpp:223-227."""
    out.write(CSV_HEADER + "\n")
    write_csv_rows(out, rep)


def csv_string(rep: BenchReport) -> str:
    buf = io.StringIO()
    write_csv(buf, rep)
    return buf.getvalue()

"""The paper's comparison (RSOC vs Çatalyürek: colours, rounds, barriers,
conflicts, time) on the device, with the reference's own runs of both on the
host cores beside it.  Tooling only; prints one JSON line per (config, side,
algorithm).
    python tools/compare_algorithms.py --configs er tri stencil rmat24
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["er", "tri", "stencil", "rmat24"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ref-runs", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    from oracle import oracle
    oracle.build()
    threads = os.cpu_count() or 1
    for cfg in args.configs:
        off, cols = graphs.make_config(cfg, "cuda")
        n, m = off.numel() - 1, cols.numel()
        g = gcol.Graph.from_device(off, cols)
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        for name, fn in (("rsoc", gcol.color_rsoc), ("catalyurek", gcol.color_catalyurek)):
            fn(g, 1, colors_out=out)
            st = [fn(g, 1, colors_out=out).stats for _ in range(args.reps)]
            print(json.dumps({
                "config": cfg, "side": "b200", "algorithm": name,
                "colors": sorted(s.num_colors for s in st), "rounds": [s.rounds for s in st],
                "barrier_events": st[-1].barrier_events,
                "conflicts_total": [s.conflicts_total for s in st],
                "ms": [round(s.wall_time_ns / 1e6, 3) for s in st],
                "GEps_best": round(m / min(s.wall_time_ns for s in st), 2)}), flush=True)
        if args.ref_runs > 0 and oracle.ref_available():
            R = oracle.RefGraph.from_csr(off.cpu().numpy(), cols.cpu().numpy())
            for name in ("rsoc", "catalyurek"):
                rs = [R.color(name, threads)[1] for _ in range(args.ref_runs)]
                print(json.dumps({
                    "config": cfg, "side": f"reference@{threads}thr", "algorithm": name,
                    "colors": sorted(r["num_colors"] for r in rs),
                    "rounds": [r["rounds"] for r in rs],
                    "barrier_events": rs[-1]["barrier_events"],
                    "conflicts_total": [r["conflicts_total"] for r in rs],
                    "ms": [round(r["wall_time_ns"] / 1e6, 1) for r in rs],
                    "GEps_best": round(m / min(r["wall_time_ns"] for r in rs), 3)}), flush=True)
            del R
        del g, off, cols
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

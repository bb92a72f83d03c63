"""A/B of the K1 variants on resident BASELINE graphs (tooling only).
    python tools/k1_ab.py [configs...] [--runs R] [--variants 0,3]
k1_wide: 1 narrow k1_pipe, 2 wide k1_pipe, 3 K1W (waiting pass), 0 auto.
Prints one JSON line per (config, variant): colours, rounds, K1 / total ms
(medians), pairs logged, and the device verification of every run.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["tri", "er", "stencil"])
    ap.add_argument("--runs", type=int, default=7)
    ap.add_argument("--variants", default="0,3")
    a = ap.parse_args()
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    for cfg in a.configs:
        off, cols = graphs.make_config(cfg, "cuda")
        g = gcol.Graph.from_device(off, cols)
        m = cols.numel()
        out = torch.empty(off.numel() - 1, dtype=torch.int32, device="cuda")
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > L2, as bench.py
        for var in [int(x) for x in a.variants.split(",")]:
            opt = gcol.ParallelOptions(k1_wide=var)
            rows = []
            for i in range(a.runs + 1):
                flush.fill_(1)
                r = gcol.color_rsoc(g, 1, opt, colors_out=out)
                rep = gcol.verify_report(g, out.cpu().numpy())[0]
                rep = (rep.violations, rep.uncolored, rep.out_of_bound)
                if i == 0:
                    continue  # warm-up (graph instantiation)
                rows.append((r.stats.num_colors, r.stats.rounds, r.stats.initial_pass_ns / 1e6,
                             r.stats.wall_time_ns / 1e6, r.stats.pairs_logged,
                             r.stats.round1_candidates, r.stats.k1_gathers, rep))
            k1 = statistics.median(x[2] for x in rows)
            tot = statistics.median(x[3] for x in rows)
            print(json.dumps({
                "config": cfg, "k1_wide": var, "k1w_cfg": os.environ.get("GCOL_K1W_CFG", ""), "colors": [x[0] for x in rows],
                "rounds": [x[1] for x in rows], "k1_ms": round(k1, 4), "total_ms": round(tot, 4),
                "ge_s": round(m / tot / 1e6, 2), "pairs": [x[4] for x in rows],
                "cand": [x[5] for x in rows], "gathers": rows[0][6],
                "verify": str(rows[-1][7])}), flush=True)
        g.release()


if __name__ == "__main__":
    main()

"""Colour-quality / speed sweep on the GPU box (not part of the product).

For each BASELINE config: the reference's RSOC colour count on the host cores
(median of --ref-runs), serial First-Fit, and our device runs under every
priority rule x K1 residency.  Prints one JSON line per measurement.
    python tools/sweep.py --configs er tri stencil rmat24
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["er", "tri", "stencil", "rmat24"])
    ap.add_argument("--rules", nargs="+", default=["id_low", "id_high", "degree_id", "ordered"])
    ap.add_argument("--bps", nargs="+", type=int, default=[0, 2, 1])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref-runs", type=int, default=3)
    ap.add_argument("--read-all", action="store_true")
    ap.add_argument("--mega", nargs="+", type=int, default=[0])
    ap.add_argument("--scale-down", type=int, default=0)
    args = ap.parse_args()
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    from oracle import oracle
    oracle.build()
    threads = os.cpu_count()
    for cfg in args.configs:
        t0 = time.time()
        off, cols = graphs.make_config(cfg, "cuda", scale_down=args.scale_down)
        torch.cuda.synchronize()
        gen_s = time.time() - t0
        g = gcol.Graph.from_device(off, cols)
        n, m = off.numel() - 1, cols.numel()
        rec = {"config": cfg, "n": n, "m": m, "max_degree": g.max_degree(), "gen_s": gen_s}
        if args.ref_runs > 0 and oracle.ref_available():
            t0 = time.time()
            R = oracle.RefGraph.from_csr(off.cpu().numpy(), cols.cpu().numpy())
            rec["ref_build_s"] = time.time() - t0
            ff = R.first_fit_sequential()
            rec["serial_ff"] = int(len(set(ff.tolist())))
            rs = [R.color("rsoc", threads)[1] for _ in range(args.ref_runs)]
            rec["ref_rsoc_colors"] = sorted(r["num_colors"] for r in rs)
            rec["ref_rsoc_ms"] = [r["wall_time_ns"] / 1e6 for r in rs]
            rec["ref_rounds"] = [r["rounds"] for r in rs]
            rec["threads"] = threads
            del R
        print(json.dumps(rec), flush=True)
        for rule, bps, mega in [(r, b, mg) for r in args.rules for b in args.bps for mg in args.mega]:
                opt = gcol.ParallelOptions(priority=gcol.Priority[rule], k1_blocks_per_sm=bps,
                                           k1_read_all=args.read_all, k1_split_min_degree=mega,
                                           k1_wide=bps)
                out = torch.empty(n, dtype=torch.int32, device="cuda")
                gcol.color_rsoc(g, 1, opt, colors_out=out)  # warm
                res = []
                for _ in range(args.reps):
                    r = gcol.color_rsoc(g, 1, opt, colors_out=out).stats
                    res.append(r)
                print(json.dumps({
                    "config": cfg, "rule": rule, "bps": bps, "mega": mega,
                    "colors": [r.num_colors for r in res], "rounds": [r.rounds for r in res],
                    "ms": [round(r.wall_time_ns / 1e6, 4) for r in res],
                    "k1_ms": [round(r.initial_pass_ns / 1e6, 4) for r in res],
                    "GEps": round(m / (min(r.wall_time_ns for r in res)), 2),
                    "pairs": res[-1].pairs_logged, "cand": res[-1].round1_candidates,
                    "conflicts": res[-1].conflicts_total,
                    "cpr_head": res[-1].conflicts_per_round[:8]}), flush=True)
        del g, off, cols
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""Class-split vs k1_pipe probe on one config (tooling only).
    python tools/class_probe.py rmat24 [runs] [k1_wide ...]
Prints per run: colours, rounds, device ms (total / initial pass / heavy
pass), logged pairs, round-1 candidates, conflicts per round; the last run of
each variant is checked by the oracle's verify_coloring (CPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    from oracle import oracle
    cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    variants = [int(x) for x in sys.argv[3:]] or [0]
    off, cols = graphs.make_config(cfg, "cuda")
    g = gcol.Graph.from_device(off, cols)
    n = off.numel() - 1
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for w in variants:
        opt = gcol.ParallelOptions(k1_wide=w)
        gcol.color_rsoc(g, 1, opt, colors_out=out)  # warm-up (plans, graphs)
        for i in range(runs):
            flush.fill_(1)
            r = gcol.color_rsoc(g, 1, opt, colors_out=out)
            s = r.stats
            print(f"{cfg} k1_wide={w} colors {s.num_colors} rounds {s.rounds} "
                  f"ms {s.wall_time_ns / 1e6:.3f} k1 {s.initial_pass_ns / 1e6:.3f} "
                  f"heavy {s.heavy_pass_ns / 1e6:.3f} (rows {s.heavy_rows}) "
                  f"pairs {s.pairs_logged} cand {s.round1_candidates} "
                  f"gathers {s.k1_gathers} cpr {list(s.conflicts_per_round[:10])}", flush=True)
        if os.environ.get("PROBE_VERIFY", "1") == "1":
            t0 = time.time()
            c = out.cpu().numpy()
            o = oracle.CSR(off.cpu().numpy(), cols.cpu().numpy())
            bad = oracle.verify_coloring(o, c)
            deg = np.diff(off.cpu().numpy())
            ok = len(bad) == 0 and (c >= 0).all() and (c <= deg).all()
            print(f"  oracle verify: {'OK' if ok else 'FAIL'} ({len(bad)} violations, "
                  f"{time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    main()

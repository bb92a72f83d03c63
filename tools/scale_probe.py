"""Heavy-pass variants across R-MAT scales (tooling): default (waiting, short poll
budget), exact waiting (k1_wide 6), speculative (k1_wide 5); medians of 5 runs.
    python tools/scale_probe.py 18 20 22"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    for sc in [int(x) for x in sys.argv[1:]] or [18, 20, 22]:
        off, cols = graphs.rmat(sc, 16, 0.57, 0.19, 0.19, 1, "cuda")
        g = gcol.Graph.from_device(off, cols)
        out = torch.empty(off.numel() - 1, dtype=torch.int32, device="cuda")
        for name, w in (("default", 0), ("exact", 6), ("speculative", 5)):
            opt = gcol.ParallelOptions(k1_wide=w)
            gcol.color_rsoc(g, 1, opt, colors_out=out)
            rs = [gcol.color_rsoc(g, 1, opt, colors_out=out).stats for _ in range(5)]
            print(f"scale {sc} {name:12s} ms {statistics.median(s.wall_time_ns for s in rs) / 1e6:7.3f} "
                  f"colours {sorted(s.num_colors for s in rs)} rounds {sorted(s.rounds for s in rs)}", flush=True)


if __name__ == "__main__":
    main()

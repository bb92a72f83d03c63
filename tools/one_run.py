"""One color_rsoc run of a BASELINE config on a resident graph (for ncu
launch lists; GCOL_EAGER=1 makes the round kernels visible).  Tooling only.
    python tools/one_run.py rmat24
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    cfg = sys.argv[1] if len(sys.argv) > 1 else "tri"
    off, cols = graphs.make_config(cfg, "cuda")
    g = gcol.Graph.from_device(off, cols)
    out = torch.empty(off.numel() - 1, dtype=torch.int32, device="cuda")
    r = gcol.color_rsoc(g, 1, colors_out=out)
    print(cfg, "colors", r.stats.num_colors, "rounds", r.stats.rounds,
          "ms", r.stats.wall_time_ns / 1e6, "cpr", r.stats.conflicts_per_round[:12], flush=True)


if __name__ == "__main__":
    main()

"""Per-tile timestamps of K1W (GCOL_K1W_TRACE, tooling): runs a config a few
times on a resident graph, the last run's {start, end} ns per 32-row tile
land in the file GCOL_K1W_TRACE names.
    GCOL_K1W_TRACE=gpurun_out/trace_tri.bin python tools/k1w_trace.py tri
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
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(4):
        flush.fill_(1)
        r = gcol.color_rsoc(g, 1, colors_out=out)
    print(cfg, "k1_ms", r.stats.initial_pass_ns / 1e6, "colors", r.stats.num_colors, flush=True)


if __name__ == "__main__":
    main()

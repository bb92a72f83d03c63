"""K1HW exactness probe (tooling): with the waiting heavy pass the class-split
colouring must equal sequential First-Fit in the order "heavy rows ascending,
then light rows ascending" bit for bit (checked with the oracle's
first_fit_sequential on the relabelled graph).
    GCOL_K1H_V=3 python tools/hw_exact.py [scale ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def class_order_first_fit(off, cols, T=64):
    import numpy as np
    from oracle import oracle
    n = off.size - 1
    deg = np.diff(off)
    heavy = deg >= T
    order = np.concatenate([np.nonzero(heavy)[0], np.nonzero(~heavy)[0]])
    newid = np.empty(n, np.int64)
    newid[order] = np.arange(n)
    rows = np.repeat(np.arange(n), deg)
    r2, c2 = newid[rows], newid[cols]
    k = np.lexsort((c2, r2))
    off2 = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r2, minlength=n), out=off2[1:])
    ff = oracle.first_fit_sequential(oracle.CSR(off2, c2[k].astype(np.int32)))
    return ff[newid]


def main():
    import numpy as np
    import torch
    from paper_1505_04086_b200 import gcol, graphs
    from oracle import oracle
    scales = [int(x) for x in sys.argv[1:]] or [16, 18, 20]
    for sc in scales:
        off, cols = graphs.rmat(sc, 16, 0.57, 0.19, 0.19, sc, "cuda")
        g = gcol.Graph.from_device(off, cols)
        off_np, cols_np = off.cpu().numpy(), cols.cpu().numpy()
        want = class_order_first_fit(off_np, cols_np)
        for it in range(3):
            r = gcol.color_rsoc(g, 1)
            s = r.stats
            same = np.array_equal(r.coloring, want)
            bad = oracle.verify_coloring(oracle.CSR(off_np, cols_np), r.coloring)
            print(f"scale {sc} run {it}: colours {s.num_colors} (class-order FF {int(want.max()) + 1}) rounds {s.rounds} "
                  f"pairs {s.pairs_logged} heavy rows {s.heavy_rows} ms {s.wall_time_ns / 1e6:.3f} "
                  f"heavy {s.heavy_pass_ns / 1e6:.3f} exact {same} violations {len(bad)}", flush=True)


if __name__ == "__main__":
    main()

"""Where the end-to-end (host CSR) time goes: raw pinned H2D bandwidth and
the wall time of each C-ABI call (create / color / destroy).  Tooling only.
    python tools/e2e_probe.py --configs tri rmat24
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["tri"])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_1505_04086_b200 import _lib, gcol, graphs
    for cfg in args.configs:
        off, cols = graphs.make_config(cfg, "cuda")
        n, m = off.numel() - 1, cols.numel()
        h_off = off.cpu().pin_memory()
        h_cols = cols.cpu().pin_memory()
        h_out = torch.empty(n, dtype=torch.int32).pin_memory()
        d = torch.empty_like(cols)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            d.copy_(h_cols, non_blocking=True)
        torch.cuda.synchronize()
        bw = args.reps * 4 * m / (time.perf_counter() - t0) / 1e9
        del d
        copt = gcol.ParallelOptions().to_c(1)
        st = _lib.Stats()
        rows = []
        for it in range(args.reps + 1):
            h = C.c_void_p()
            t = [time.perf_counter()]
            assert _lib.LIB.gcol_cuda_graph_create(C.c_void_p(h_off.data_ptr()),
                                                   C.c_void_p(h_cols.data_ptr()), n, m,
                                                   _lib.GCOL_MEM_HOST, -1, C.byref(h)) == 0
            t.append(time.perf_counter())
            assert _lib.LIB.gcol_cuda_color_rsoc(h, C.byref(copt), C.c_void_p(h_out.data_ptr()),
                                                 _lib.GCOL_MEM_HOST, C.byref(st)) == 0
            t.append(time.perf_counter())
            assert _lib.LIB.gcol_cuda_color_rsoc(h, C.byref(copt), C.c_void_p(h_out.data_ptr()),
                                                 _lib.GCOL_MEM_HOST, C.byref(st)) == 0
            t.append(time.perf_counter())
            _lib.LIB.gcol_cuda_graph_destroy(h)
            t.append(time.perf_counter())
            rows.append([round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])])
        one = []
        for it in range(args.reps + 1):
            t0 = time.perf_counter()
            r = gcol.color_rsoc_csr(h_off, h_cols, 1, colors_out=h_out)
            one.append((round((time.perf_counter() - t0) * 1e3, 3),
                        round(r.stats.wall_time_ns / 1e6, 3), round(r.stats.initial_pass_ns / 1e6, 3),
                        r.stats.rounds))
        print({"config": cfg, "one_call (wall ms, device ms from K1 start, k1 ms, rounds)": one})
        print({"config": cfg, "n": n, "m": m, "h2d_GBps_pinned": round(bw, 1),
               "h2d_ms_ideal": round((8 * (n + 1) + 4 * m) / bw / 1e6, 3),
               "device_ms": st.wall_time_ns / 1e6,
               "create/color1/color2/destroy ms": rows}, flush=True)


if __name__ == "__main__":
    main()

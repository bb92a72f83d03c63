"""Alternating one-call vs three-call end-to-end timings (medians).  Tooling only."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1505_04086_b200 import _lib, gcol, graphs
    reps = int(os.environ.get("REPS", "10"))
    for cfg in sys.argv[1:] or ["tri", "er"]:
        off, cols = graphs.make_config(cfg, "cuda")
        n, m = off.numel() - 1, cols.numel()
        h_off, h_cols = off.cpu().pin_memory(), cols.cpu().pin_memory()
        h_out = torch.empty(n, dtype=torch.int32).pin_memory()
        copt = gcol.ParallelOptions().to_c(1)
        st = _lib.Stats()
        po, pc, pout = (C.c_void_p(t.data_ptr()) for t in (h_off, h_cols, h_out))

        def one():
            assert _lib.LIB.gcol_cuda_color_rsoc_csr(po, pc, n, m, -1, C.byref(copt), pout,
                                                     C.byref(st)) == 0

        def three():
            h = C.c_void_p()
            assert _lib.LIB.gcol_cuda_graph_create(po, pc, n, m, _lib.GCOL_MEM_HOST, -1, C.byref(h)) == 0
            assert _lib.LIB.gcol_cuda_color_rsoc(h, C.byref(copt), pout, _lib.GCOL_MEM_HOST, C.byref(st)) == 0
            _lib.LIB.gcol_cuda_graph_destroy(h)

        one(); three()
        t1, t3 = [], []
        for _ in range(reps):
            a = time.perf_counter(); one(); t1.append(time.perf_counter() - a)
            a = time.perf_counter(); three(); t3.append(time.perf_counter() - a)
        print(cfg, "one-call ms median %.3f min %.3f | three-call median %.3f min %.3f" % (
            1e3 * statistics.median(t1), 1e3 * min(t1), 1e3 * statistics.median(t3), 1e3 * min(t3)),
            flush=True)


if __name__ == "__main__":
    main()

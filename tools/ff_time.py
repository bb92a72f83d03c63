import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1505_04086_b200 import gcol, graphs
for name, sd in (("tri", 0), ("stencil", 0), ("rmat24", 4)):
    off, cols = graphs.make_config(name, "cuda", scale_down=sd)
    g = gcol.Graph.from_device(off, cols)
    gcol.first_fit_sequential(g)
    t = time.perf_counter(); ff = gcol.first_fit_sequential(g); dt = time.perf_counter() - t
    print(name, "max_degree", g.max_degree(), "first_fit_sequential wall ms %.2f" % (dt * 1e3), "colors", len(set(ff.tolist())), flush=True)

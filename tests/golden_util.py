"""Loader for the reference-generated fixtures in tests/golden/."""
import os
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def coloring_fixtures():
    z = np.load(os.path.join(GOLDEN, "ref_coloring.npz"))
    names = [str(x) for x in z["names"]]
    cases = {}
    for name in names:
        cases[name] = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(name + "/")}
    return cases


@lru_cache(maxsize=None)
def lockstep_fixtures():
    z = np.load(os.path.join(GOLDEN, "ref_lockstep.npz"))
    out = {}
    for k in z.files:
        name, field = k.split("/", 1)
        out.setdefault(name, {})[field] = z[k]
    return out

"""CPU: the C-ABI library, the host-side mirror of the reference interface,
and the synthetic generators.  No compute calls are made without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from tests.golden_util import coloring_fixtures

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "gcol_cuda.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(gcol_cuda_\w+)\(", src, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1505_04086_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(_lib.LIB, s), f"{s} declared in include/gcol_cuda.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert _lib.LIB.gcol_cuda_abi_version() == 2


def test_struct_layouts_match_header():
    """Field count / order of the ctypes mirrors against the C header."""
    from paper_1505_04086_b200 import _lib
    src = open(os.path.join(REPO, "include", "gcol_cuda.h")).read()

    def fields(struct_name):
        body = re.search(r"typedef struct \{((?:(?!typedef struct).)*?)\} " + struct_name + ";", src,
                         re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        return re.findall(r"\b(\w+)(?:\[\d+\])?;", body)

    assert fields("gcol_cuda_options") == [f for f, _ in _lib.Options._fields_]
    assert fields("gcol_cuda_stats") == [f for f, _ in _lib.Stats._fields_]
    assert fields("gcol_cuda_verify_report") == [f for f, _ in _lib.VerifyReport._fields_]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_no_device_fails_loudly():
    from paper_1505_04086_b200 import gcol
    g = gcol.build_graph([(0, 1)], 2)
    with pytest.raises(gcol.NoDeviceError):
        gcol.color_rsoc(g, 1)
    assert gcol.device_count() == 0


@pytest.mark.parametrize("name", [k for k, v in coloring_fixtures().items() if "edges" in v])
def test_build_graph_matches_reference(name):
    """gcol.build_graph (host numpy) == the reference's build_graph CSR."""
    from paper_1505_04086_b200 import gcol
    case = coloring_fixtures()[name]
    g = gcol.build_graph(case["edges"], int(case["n"][0]))
    assert np.array_equal(g.offsets(), case["off"])
    assert np.array_equal(g.adjacency(), case["cols"])
    g.validate()
    assert g.max_degree() == (int(np.diff(case["off"]).max()) if case["off"].size > 1 else 0)


def test_build_graph_examples_and_errors():  # SPEC.md graph-core examples, graph.hpp:100-104
    from paper_1505_04086_b200 import gcol
    g = gcol.build_graph([], 0)
    assert g.num_vertices() == 0 and g.max_degree() == 0
    g = gcol.build_graph([(0, 1), (1, 0), (1, 1)], 2)
    assert g.num_edges() == 1 and g.max_degree() == 1
    g = gcol.build_graph([(0, 1), (1, 2), (2, 0)], 3)
    assert all(g.degree(v) == 2 for v in range(3))
    assert g.degree(0) == 2 and list(g.neighbors(1)) == [0, 2]
    with pytest.raises(gcol.input_error):
        gcol.build_graph([(0, 5)], 3)
    with pytest.raises(gcol.input_error):
        g.degree(3)


def test_graph_validate_detects_corruption():  # graph.hpp:50-77
    from paper_1505_04086_b200 import gcol
    bad = [
        (np.array([0, 1, 1]), np.array([1])),            # one direction only
        (np.array([0, 1, 2]), np.array([0, 0])),         # self loop
        (np.array([0, 2, 3, 4]), np.array([2, 1, 0, 0])),  # unsorted row
        (np.array([0, 1, 2]), np.array([1, 5])),         # out of range
    ]
    for off, cols in bad:
        with pytest.raises(gcol.input_error):
            gcol.Graph(off, cols).validate()


def test_generators_valid_and_deterministic():
    from paper_1505_04086_b200 import gcol, graphs
    for f in (lambda: graphs.erdos_renyi(3000, 16, 5), lambda: graphs.tri_mesh(30, 20, 5),
              lambda: graphs.stencil27(9, 8, 7, 5), lambda: graphs.rmat(11, 16, .57, .19, .19, 5)):
        o1, c1 = f()
        o2, c2 = f()
        assert torch.equal(o1, o2) and torch.equal(c1, c2)
        g = gcol.Graph(o1.numpy(), c1.numpy())
        g.validate()
    off, cols = graphs.tri_mesh(40, 40, 1)
    assert cols.numel() == 2 * (39 * 40 * 2 + 39 * 39) and int(torch.diff(off).max()) == 6
    off, cols = graphs.stencil27(10, 10, 10, 1)
    assert int(torch.diff(off).max()) == 26
    # 13 forward directions on a 10^3 grid: 2*(3*9*100 + 6*9*9*10 + 4*9*9*9)
    assert cols.numel() == 2 * (3 * 900 + 6 * 810 + 4 * 729)


def test_rmat_bucketed_builder_is_the_same_csr():
    """The memory-lean bucketed R-MAT builder (used above 2^28 samples, i.e.
    BASELINE configs[4], scale 27) yields exactly the canonical CSR of the
    direct build, for several bucket counts and chunk sizes."""
    from paper_1505_04086_b200 import graphs
    o1, c1 = graphs.rmat(12, 16, .57, .19, .19, 7, lean=False)
    perm = graphs.random_permutation(1 << 12, 7, "cpu")
    for nb, chunk in ((1, 1 << 20), (8, 1 << 11), (64, 5000)):
        o2, c2 = graphs._rmat_csr_bucketed(12, 16 << 12, .57, .19, .19, 7, perm, "cpu", chunk,
                                           nbuckets=nb)
        assert torch.equal(o1, o2) and torch.equal(c1, c2)


def test_generators_reference_build_parity(oracle_mod):
    """Our torch CSR construction (csr_from_edges and the bucketed builder)
    == the reference's build_graph (graph.hpp:98-138) fed the SAME raw pair
    multiset: self-loops, duplicates in both orientations and isolated ids
    included, so a dedup, loop or sort bug cannot hide."""
    from paper_1505_04086_b200 import graphs
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")

    def ref_csr(u, v, n):
        e = torch.stack([u, v], 1).numpy()
        csr = oracle_mod.RefGraph.from_edges(e, n).csr()
        return csr.off.astype(np.int64), csr.cols.astype(np.int32)

    cases = []
    u, v = graphs.rmat_pairs(11, 16, .57, .19, .19, 3)
    cases.append(("rmat", u, v, 1 << 11))
    u, v = graphs.erdos_renyi_pairs(3000, 9.0, 5)
    cases.append(("er", u, v, 3000))
    g = torch.Generator().manual_seed(9)
    u = torch.randint(0, 50, (4000,), generator=g)
    v = torch.randint(0, 50, (4000,), generator=g)
    u[::7] = v[::7]                                   # explicit self-loops
    u = torch.cat([u, v[:500]]); v = torch.cat([v, u[:500]])  # reversed duplicates
    cases.append(("dense-dups", u, v, 64))            # ids 50..63 isolated
    for name, u, v, n in cases:
        assert bool((u == v).any()), name             # the multiset holds loops
        ro, rc = ref_csr(u, v, n)
        off, cols = graphs.csr_from_edges(u, v, n)
        assert np.array_equal(off.numpy(), ro), name
        assert np.array_equal(cols.numpy(), rc), name
    # the rmat generator's own path (direct and bucketed) == build_graph of its pairs
    u, v = graphs.rmat_pairs(11, 16, .57, .19, .19, 3)
    ro, rc = ref_csr(u, v, 1 << 11)
    for lean in (False, True):
        off, cols = graphs.rmat(11, 16, .57, .19, .19, 3, lean=lean)
        assert np.array_equal(off.numpy(), ro) and np.array_equal(cols.numpy(), rc), lean
    off, cols = graphs.erdos_renyi(3000, 9.0, 5)
    ro, rc = ref_csr(*graphs.erdos_renyi_pairs(3000, 9.0, 5), 3000)
    assert np.array_equal(off.numpy(), ro) and np.array_equal(cols.numpy(), rc)

"""GPU: the multi-GPU building blocks of the C ABI (k1_range, detect_range,
round_list, scatter_colors) through DeviceOps, with P logical partitions
emulated on one device: each partition has its own replica, and the test
performs the exchange steps of dist.color_rsoc_distributed by hand.  (The
collective orchestration itself is covered over gloo in tests/test_dist.py;
ranks are never co-scheduled as interdependent kernels on one GPU.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1505_04086_b200 import dist as gdist, gcol, graphs  # noqa: E402


def emulate(g, n, P):
    ops = gdist.DeviceOps(g)
    parts = gdist.partition(n, P)
    reps = [torch.full((n,), -1, dtype=torch.int32, device="cuda") for _ in range(P)]
    for r, (lo, hi) in enumerate(parts):
        ops.k1_range(reps[r], lo, hi)
    for r in range(P):  # all-gather of owned slices
        for q, (lo, hi) in enumerate(parts):
            if q != r:
                reps[r][lo:hi] = reps[q][lo:hi]
    work = [ops.detect_range(reps[r], lo, hi) for r, (lo, hi) in enumerate(parts)]
    rounds = 0
    while True:
        rec = [ops.round_list(reps[r], work[r]) for r in range(P)]
        vals = [reps[r][rec[r].long()] for r in range(P)]
        for r in range(P):
            for q in range(P):
                if q != r and rec[q].numel():
                    ops.scatter(reps[r], rec[q], vals[q])
        rounds += 1
        if sum(x.numel() for x in rec) == 0:
            break
        work = rec
        assert rounds < 1000
    return reps, rounds


@pytest.mark.parametrize("P", [1, 2, 4])
def test_partitioned_blocks(P):
    off, cols = graphs.erdos_renyi(60_000, 16, 11, "cuda")
    n = off.numel() - 1
    g = gcol.Graph.from_device(off, cols)
    reps, rounds = emulate(g, n, P)
    for r in range(1, P):
        assert torch.equal(reps[0], reps[r])
    hg = gcol.Graph(off.cpu().numpy(), cols.cpu().numpy())
    c = reps[0].cpu().numpy()
    assert gcol.verify_coloring(hg, c).ok()
    assert (c >= 0).all() and (c <= np.diff(hg.offsets())).all()
    assert gcol.count_colors(c) <= hg.max_degree() + 1


def test_k1_range_matches_full_on_one_partition():
    off, cols = graphs.tri_mesh(300, 300, 3, "cuda")
    n = off.numel() - 1
    g = gcol.Graph.from_device(off, cols)
    ops = gdist.DeviceOps(g)
    colors = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    ops.k1_range(colors, 0, n)
    assert (colors >= 0).all()
    with pytest.raises(gcol.input_error):
        ops.k1_range(colors, 3, n)  # ranges start on 256-id chunk boundaries


def emulate_push(off, cols, n, P, priority=gcol.Priority.degree_id):
    """Push mode with P logical ranks on one device, run one after another
    (no rank waits on another): rank r's handle pushes every colour it
    commits into the other ranks' replicas through their device pointers,
    the same stores that go over NVLink between GPUs."""
    # no rank may wait on another here (they run one after another): the
    # waiting initial pass is told not to wait (k1_wait_polls < 0), so every
    # in-flight read of another rank's row is logged, as optimistic RSOC does
    opt = gcol.ParallelOptions(priority=priority, k1_wait_polls=-1)
    ops = [gdist.DeviceOps(gcol.Graph.from_device(off, cols), priority=int(priority), opt=opt)
           for _ in range(P)]
    reps = [torch.full((n,), -1, dtype=torch.int32, device="cuda") for _ in range(P)]
    ptrs = [t.data_ptr() for t in reps]
    for r in range(P):
        ops[r].partition(r, P, ptrs)
    for r in range(P):
        ops[r].k1_owned(reps[r])
    torch.cuda.synchronize()
    every = torch.cat([ops[r].candidates(reps[r]) for r in range(P)])
    own = gdist.owner_of(every.long(), P)
    work = [torch.unique(every[own == r]).to(torch.int32) for r in range(P)]
    cand = sum(w.numel() for w in work)
    rounds = 0
    while True:
        rec = [ops[r].round_list(reps[r], work[r]) for r in range(P)]
        rounds += 1
        if sum(x.numel() for x in rec) == 0:
            break
        work = rec
        assert rounds < 1000
    return reps, rounds, cand


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_push_mode_partitions(P):
    off, cols = graphs.erdos_renyi(80_000, 16, 12, "cuda")
    n = off.numel() - 1
    reps, rounds, cand = emulate_push(off, cols, n, P)
    for r in range(1, P):
        assert torch.equal(reps[0], reps[r]), "replicas diverged"
    hg = gcol.Graph(off.cpu().numpy(), cols.cpu().numpy())
    c = reps[0].cpu().numpy()
    assert gcol.verify_coloring(hg, c).ok()
    assert (c >= 0).all() and (c <= np.diff(hg.offsets())).all()
    assert gcol.count_colors(c) <= hg.max_degree() + 1


def test_push_mode_skewed_graph():
    """Hubs split into pieces and dynamic sub-tiles under the partition."""
    off, cols = graphs.make_config("rmat24", "cuda", scale_down=7)
    n = off.numel() - 1
    reps, rounds, cand = emulate_push(off, cols, n, 4)
    for r in range(1, 4):
        assert torch.equal(reps[0], reps[r])
    hg = gcol.Graph(off.cpu().numpy(), cols.cpu().numpy())
    c = reps[0].cpu().numpy()
    assert gcol.verify_coloring(hg, c).ok()
    assert (c <= np.diff(hg.offsets())).all()


def test_push_mode_one_rank_k1w_is_serial_ff():
    """Bounded degree under the partition (world of one): the owned-chunk
    initial pass is K1W, which waits instead of logging -- serial First-Fit,
    no candidates, one empty round."""
    off, cols = graphs.erdos_renyi(50_000, 12, 4, "cuda")
    n = off.numel() - 1
    hg = gcol.Graph(off.cpu().numpy(), cols.cpu().numpy())
    assert hg.max_degree() <= 63
    ops = gdist.DeviceOps(gcol.Graph.from_device(off, cols), priority=int(gcol.Priority.degree_id))
    colors = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    ops.partition(0, 1, [colors.data_ptr()])
    ops.k1_owned(colors)
    torch.cuda.synchronize()
    assert ops.candidates(colors).numel() == 0
    from oracle import oracle as oracle_mod  # the CPU checker, not the device First-Fit
    oracle_mod.build()
    ff = oracle_mod.first_fit_sequential(oracle_mod.CSR(hg.offsets(), hg.adjacency()))
    assert np.array_equal(colors.cpu().numpy(), ff)


def emulate_push_concurrent(off, cols, n, P, priority=gcol.Priority.degree_id):
    """Push mode with P logical ranks running AT THE SAME TIME on one device:
    one host thread and one stream (handle) per rank, each rank's initial
    pass on 1/P of the SMs (GCOL_K1_WAIT_BPS), so its pushes, the other
    ranks' stale remote reads and the cross-rank K1W waits interleave as
    they would between GPUs.  Rounds run concurrently too; a round ends when
    every rank's recolours (and pushes) are done."""
    import threading
    opt = gcol.ParallelOptions(priority=priority)
    ops = [gdist.DeviceOps(gcol.Graph.from_device(off, cols), priority=int(priority), opt=opt)
           for _ in range(P)]
    reps = [torch.full((n,), -1, dtype=torch.int32, device="cuda") for _ in range(P)]
    ptrs = [t.data_ptr() for t in reps]
    for r in range(P):
        ops[r].partition(r, P, ptrs)
    torch.cuda.synchronize()

    def all_ranks(fn):
        out, errs = [None] * P, []

        def run(r):
            try:
                out[r] = fn(r)
            except Exception as e:  # noqa: BLE001
                errs.append(e)
        th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
        assert not any(t.is_alive() for t in th), "a rank hung"
        assert not errs, errs
        torch.cuda.synchronize()
        return out

    all_ranks(lambda r: ops[r].k1_owned(reps[r]))
    every = torch.cat([ops[r].candidates(reps[r]) for r in range(P)])
    own = gdist.owner_of(every.long(), P)
    work = [torch.unique(every[own == r]).to(torch.int32) for r in range(P)]
    rounds = 0
    while True:
        rec = all_ranks(lambda r: ops[r].round_list(reps[r], work[r]))
        rounds += 1
        if sum(x.numel() for x in rec) == 0:
            break
        work = rec
        assert rounds < 1000
    return reps, rounds


@pytest.mark.parametrize("P", [2, 4])
def test_push_mode_concurrent_ranks(P, monkeypatch):
    import os
    occ = 6  # K1W's resident CTAs per SM (kWaitMinBlocks)
    monkeypatch.setenv("GCOL_K1_WAIT_BPS", str(max(1, occ // P)))
    off, cols = graphs.erdos_renyi(120_000, 16, 21, "cuda")
    n = off.numel() - 1
    reps, rounds = emulate_push_concurrent(off, cols, n, P)
    for r in range(1, P):
        assert torch.equal(reps[0], reps[r]), "replicas diverged"
    hg = gcol.Graph(off.cpu().numpy(), cols.cpu().numpy())
    c = reps[0].cpu().numpy()
    from oracle import oracle as oracle_mod
    oracle_mod.build()
    o = oracle_mod.CSR(hg.offsets(), hg.adjacency())
    assert oracle_mod.verify_coloring(o, c) == []
    assert (c >= 0).all() and (c <= np.diff(hg.offsets())).all()
    del os

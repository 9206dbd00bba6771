"""Fused push exchange of the row partition on one B200.

A PartitionGroup drives G ranks of the same graph from one process: every rank's term kernel
stores x_{k+1} straight into the buffers of the ranks that read it (halo push), and a release/acquire flag barrier
separates the terms.  On one GPU the ranks run in lockstep (each rank's wait kernel is
event-ordered after every rank's signal, so no kernel spins on work not yet enqueued).  The
kernels, buffers and barrier are the ones a one-process-per-GPU run uses over NVLink.
Checked against the single-GPU solve and the reference's golden ranks."""
import numpy as np
import pytest

from conftest import load_golden

TOL64 = 1e-12

pytestmark = pytest.mark.gpu


def top_k(r, k=100):
    return np.lexsort((np.arange(r.size), -r))[:k]


def _handles(cheb, edges, G):
    return [cheb.build_device_graph(edges)[0] for _ in range(G)]


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name", ["config1", "gnp2000", "star100"])
def test_push_group_matches_single_gpu_and_reference(cheb, name, G):
    z = load_golden(name)
    single_dg, _ = cheb.build_device_graph(z["edges"])
    single = cheb.run_cpaa(single_dg, cheb.SolverConfig(rounds=39))
    hs = _handles(cheb, z["edges"], G)
    grp = cheb.PartitionGroup(hs)
    res = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=39))
    assert res.rounds == 39
    assert np.max(np.abs(res.ranks - single.ranks)) <= TOL64
    assert np.max(np.abs(res.ranks - z["cpaa39_ranks"])) <= TOL64
    k = min(100, res.ranks.size)
    assert np.array_equal(top_k(res.ranks, k), top_k(z["cpaa39_ranks"], k))
    for a, b in zip(res.trace, single.trace):  # rank-ordered trace combine
        assert a.k == b.k and a.c_k == b.c_k
        assert abs(a.S_k - b.S_k) <= 1e-9 * abs(b.S_k)
        assert abs(a.mass_T - b.mass_T) <= 1e-9 * max(1.0, abs(b.mass_T))
    again = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=39))  # barrier epochs keep counting
    assert np.array_equal(again.ranks, res.ranks)
    grp.close()
    # detached handles are single-GPU handles again
    after = cheb.run_cpaa(hs[0], cheb.SolverConfig(rounds=39))
    assert np.array_equal(after.ranks, single.ranks)


def test_push_group_hub_rows_and_eps(cheb):
    """A power-law graph with rows above the warp tile (hub chunks finalised by the second
    kernel, whose epilogue pushes too), planned by eps."""
    from paper_2112_01743_b200 import generate as Gen
    e = Gen.chung_lu_edges(1 << 15, 2.1, 2.0, 5000.0, 200_000, 9)
    single_dg, info = cheb.build_device_graph(e)
    assert info["max_degree"] > 248
    single = cheb.run_cpaa(single_dg, cheb.SolverConfig(eps=1e-10))
    for G in (2, 4):
        grp = cheb.PartitionGroup(_handles(cheb, e, G))
        res = cheb.run_cpaa(grp, cheb.SolverConfig(eps=1e-10))
        assert res.rounds == single.rounds == 39
        assert np.max(np.abs(res.ranks - single.ranks)) <= TOL64
        assert np.array_equal(top_k(res.ranks), top_k(single.ranks))
        grp.close()


@pytest.mark.parametrize("halo", [1, 0])
def test_push_group_with_column_windows(cheb, halo):
    """Partitioned ranks with the hub rows' column windows forced on (every rank's window pass
    reads the x its peers pushed, behind the term barrier): equal to the single-GPU solve
    within 1e-12 with the same top-100, fp64 and fp32, repeated solves bitwise equal."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    import ctypes as C
    lib = _lib.load()
    e = Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 20000.0, 900_000, 5)
    single_dg, info = cheb.build_device_graph(e)
    single = cheb.run_cpaa(single_dg, cheb.SolverConfig(eps=1e-10))
    try:
        assert lib.cheb_set_tuning(b"windows", 6) == 0 and lib.cheb_set_tuning(b"winsize", 2048) == 0
        assert lib.cheb_set_tuning(b"halo", halo) == 0
        for G in (2, 4):
            hs = _handles(cheb, e, G)
            grp = cheb.PartitionGroup(hs)
            res = cheb.run_cpaa(grp, cheb.SolverConfig(eps=1e-10))
            sizes = np.zeros(8, dtype=np.int64)
            assert lib.cheb_graph_view_windows(hs[0].handle, sizes.ctypes.data_as(C.POINTER(C.c_int64)),
                                               None, None, None, None, None) == 0
            assert sizes[0] == 6 and sizes[4] > 0          # the rank's view has windows
            assert np.max(np.abs(res.ranks - single.ranks)) <= TOL64
            assert np.array_equal(top_k(res.ranks), top_k(single.ranks))
            again = cheb.run_cpaa(grp, cheb.SolverConfig(eps=1e-10))
            assert np.array_equal(again.ranks, res.ranks)
            f32 = cheb.run_cpaa(grp, cheb.SolverConfig(eps=1e-10, precision=32))
            assert np.sum(np.abs(f32.ranks - single.ranks)) / np.sum(single.ranks) <= 1e-6
            grp.close()
    finally:
        lib.cheb_set_tuning(b"windows", -1)
        lib.cheb_set_tuning(b"winsize", 28672)
        lib.cheb_set_tuning(b"halo", 1)


def test_push_group_zero_rounds_and_fp32(cheb):
    z = load_golden("gnp2000")
    grp = cheb.PartitionGroup(_handles(cheb, z["edges"], 2))
    r0 = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=0))
    assert r0.rounds == 0 and np.allclose(r0.ranks, 1.0 / z["n"], rtol=0, atol=1e-15)
    r32 = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=39, precision=32))
    ref = z["cpaa39_ranks"]
    assert np.abs(r32.ranks - ref).sum() / np.abs(ref).sum() <= 1e-6
    grp.close()


def test_push_group_rejects_mixed_graphs(cheb):
    a, _ = cheb.build_device_graph(load_golden("gnp2000")["edges"])
    b, _ = cheb.build_device_graph(load_golden("config1")["edges"])
    with pytest.raises(ValueError, match="same graph"):
        cheb.PartitionGroup([a, b])


def test_peer_exchange_single_rank_ipc(cheb):
    """The one-process-per-GPU wiring at world size 1: the exchange buffers are exported as
    CUDA IPC handles and imported back, cheb_cpaa runs the partitioned solve with the push
    exchange and the device flag barrier (signal + spin-wait kernels)."""
    from paper_2112_01743_b200.distributed import PeerExchange
    z = load_golden("config1")
    dg, _ = cheb.build_device_graph(z["edges"])
    plain = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
    px = PeerExchange(dg, 0, 1)
    part = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
    assert np.max(np.abs(part.ranks - plain.ranks)) <= TOL64
    assert np.max(np.abs(part.ranks - z["cpaa39_ranks"])) <= TOL64
    px.detach()
    again = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
    assert np.array_equal(again.ranks, plain.ranks)


@pytest.mark.parametrize("name,G", [("path3", 5), ("k2", 3), ("cycle4", 4), ("star100", 8)])
def test_push_group_more_ranks_than_work(cheb, name, G):
    """Tiny graphs cut into more ranks than they have (or nearly have) rows: empty slices
    push nothing but still signal every barrier."""
    z = load_golden(name)
    single = cheb.run_cpaa(cheb.build_device_graph(z["edges"])[0], cheb.SolverConfig(rounds=39))
    grp = cheb.PartitionGroup(_handles(cheb, z["edges"], G))
    res = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=39))
    assert np.max(np.abs(res.ranks - single.ranks)) <= TOL64
    assert np.max(np.abs(res.ranks - z["cpaa39_ranks"])) <= TOL64
    grp.close()


def test_push_group_personalised(cheb):
    """A personalisation vector (T_0 = p) on a partitioned solve: the ranks index p by the
    original vertex id through their slice of the view order."""
    z = load_golden("gnp2000")
    rng = np.random.default_rng(4)
    p = rng.random(int(z["n"]))
    single = cheb.run_cpaa(cheb.build_device_graph(z["edges"])[0],
                           cheb.SolverConfig(rounds=39, personalization=p))
    for G in (2, 3):
        grp = cheb.PartitionGroup(_handles(cheb, z["edges"], G))
        res = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=39, personalization=p))
        assert np.max(np.abs(res.ranks - single.ranks)) <= TOL64
        grp.close()


def test_push_group_int64_row_pointers(cheb):
    """Partitioned solve on handles with int64 row pointers (the config-4 layout)."""
    z = load_golden("config1")
    single = cheb.run_cpaa(cheb.build_device_graph(z["edges"])[0], cheb.SolverConfig(rounds=39))
    hs = [cheb.build_device_graph(z["edges"], cheb.BuildOptions(row_ptr_64=True))[0] for _ in range(2)]
    grp = cheb.PartitionGroup(hs)
    res = cheb.run_cpaa(grp, cheb.SolverConfig(rounds=39))
    assert np.max(np.abs(res.ranks - single.ranks)) <= TOL64
    grp.close()


def test_peer_and_group_argument_errors(cheb):
    """The push-exchange entry points reject bad arguments with CHEB_INVALID_ARG."""
    import ctypes as C
    from paper_2112_01743_b200 import _lib as L
    lib = L.load()
    z = load_golden("k2")
    dg, _ = cheb.build_device_graph(z["edges"])
    out = C.c_void_p()
    assert lib.cheb_group_create((C.c_void_p * 1)(dg.handle), 0, C.byref(out)) == 4       # G < 1
    assert lib.cheb_group_create((C.c_void_p * 2)(dg.handle, dg.handle), 2, C.byref(out)) == 4  # duplicate
    buf = (C.c_ubyte * 16)()
    assert lib.cheb_peer_export(dg.handle, 2, 0, buf, 16) == 4                                # too small
    big = (C.c_ubyte * L.PEER_EXPORT_BYTES)()
    assert lib.cheb_peer_import(dg.handle, big, L.PEER_EXPORT_BYTES) == 4                     # no export yet
    assert lib.cheb_peer_export(dg.handle, 2, 5, big, L.PEER_EXPORT_BYTES) == 4               # rank >= G
    # the handle still solves as a single-GPU graph after the failed calls
    r = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=5))
    assert np.allclose(r.ranks, 0.5)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_halo_push_volume_and_bitwise_equivalence(cheb, G):
    """Halo-only push: rank r receives x_{k+1}[u] only when one of its rows has neighbour u
    (for a symmetric graph: u has a neighbour owned by r).  The stores skipped are exactly the
    ones never read, so the solve is bitwise the replicate-to-all solve; the store counts per
    rank equal a numpy recount of the masks from the partition plan."""
    import ctypes as C
    from paper_2112_01743_b200 import _lib as L
    from paper_2112_01743_b200 import generate as Gen
    from paper_2112_01743_b200.distributed import partition_plan
    lib = L.load()
    e = Gen.chung_lu_edges(1 << 15, 2.1, 2.0, 5000.0, 150_000, 4)
    hs = _handles(cheb, e, G)
    grp = cheb.PartitionGroup(hs)
    halo = cheb.run_cpaa(grp, cheb.SolverConfig(eps=1e-10))
    stores = []
    for h in hs:
        a, b = C.c_int64(), C.c_int64()
        assert lib.cheb_graph_exchange_info(h.handle, C.byref(a), C.byref(b)) == 0
        stores.append((a.value, b.value))
    assert lib.cheb_set_tuning(b"halo", 0) == 0
    try:
        full = cheb.run_cpaa(grp, cheb.SolverConfig(eps=1e-10))
    finally:
        lib.cheb_set_tuning(b"halo", 1)
    assert np.array_equal(halo.ranks, full.ranks)
    grp.close()
    # numpy recount: owner of each sorted row (block-cyclic snake partition), masks over each
    # local row's neighbours
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from multigpu_emul import block_rows, part_owner
    B = block_rows()
    g = hs[0].download()
    order, _, _ = partition_plan(g.degrees, G)
    new = np.empty(g.n, dtype=np.int64)
    new[order] = np.arange(g.n)
    rows = np.repeat(new, np.diff(g.offsets))          # sorted id of each entry's row
    owner_col = part_owner(new[g.neighbors], G, B)
    pairs = np.unique(rows * G + owner_col)            # (row, rank needing it)
    prow = pairs // G
    pr = pairs % G
    prow_owner = part_owner(prow, G, B)
    n_rows = np.bincount(part_owner(np.arange(g.n), G, B), minlength=G)
    for r in range(G):
        mine = prow_owner == r
        want_halo = int(np.count_nonzero(mine & (pr != r)))
        assert stores[r] == (want_halo, int(n_rows[r]) * (G - 1)), (r, stores[r], want_halo)
    assert sum(s[0] for s in stores) < sum(s[1] for s in stores)

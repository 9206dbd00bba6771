"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the committed
reference fixtures.  Bars (BASELINE.json north_star): CSR/degrees bit-exact; fp64 ranks
within 1e-12 max-abs and identical top-100 (FAST); BITEXACT mode bitwise; fp32 relative
L1 <= 1e-6."""
import numpy as np
import pytest

from conftest import GOLDEN_NAMES, load_golden

pytestmark = pytest.mark.gpu
C = 0.85
TOL64 = 1e-12     # fp64 max-abs (north_star)
TOL32_L1 = 1e-6   # fp32 relative L1 (north_star)


def build_kw(name):
    kw = {}
    if name == "multi":
        kw["dedup"] = False
    if name in ("drop", "nhint_drop"):
        kw["drop_isolated"] = True
    if name == "nhint_drop":
        kw["n_hint"] = 6
    return kw


def top_k(r, k=100):
    # ties broken by vertex id (stable sort on -rank)
    return np.argsort(-r, kind="stable")[:k]


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_device_csr_builder_bit_exact(cheb, name):
    z = load_golden(name)
    res = cheb.build_graph(z["edges"], cheb.BuildOptions(**build_kw(name)))
    g = res.graph
    assert g.n == int(z["n"]) and g.m == int(z["m"])
    assert np.array_equal(g.offsets, z["offsets"])
    assert np.array_equal(g.neighbors, z["neighbors"])
    assert np.array_equal(g.degrees, z["degrees"])
    assert res.duplicates_removed == int(z["duplicates_removed"])
    assert res.isolated_dropped == int(z["isolated_dropped"])
    assert g.multi == bool(z["multi"])


@pytest.mark.parametrize("row_ptr_64", [False, True])
def test_device_csr_builder_row_ptr_widths(cheb, oracle, row_ptr_64):
    e = oracle.gnp_edges(3000, 0.004, 9)
    ref = oracle.build_graph(e)
    g = cheb.build_graph(e, cheb.BuildOptions(row_ptr_64=row_ptr_64)).graph
    assert np.array_equal(g.offsets, ref.offsets) and np.array_equal(g.neighbors, ref.neighbors)


def test_device_csr_builder_errors(cheb):
    with pytest.raises(cheb.ValidationError, match="vertex 2 is isolated"):
        cheb.build_graph([[0, 1], [3, 4]])
    with pytest.raises(cheb.ValidationError, match="negative vertex id"):
        cheb.build_graph([[0, -1]])
    with pytest.raises(cheb.ValidationError):
        cheb.build_graph([[0, 1]], cheb.BuildOptions(n_hint=4))
    r = cheb.build_graph([[0, 1]], cheb.BuildOptions(n_hint=4, drop_isolated=True))
    assert r.graph.n == 2 and r.isolated_dropped == 2
    r = cheb.build_graph(np.zeros((0, 2), np.int64), cheb.BuildOptions(drop_isolated=True))
    assert r.graph.n == 0
    with pytest.raises(cheb.CapacityError):  # max id + 1 would overflow int64 (graph.cpp:25-29)
        cheb.build_graph([[0, 2**63 - 1]])
    with pytest.raises(cheb.CapacityError):
        cheb.build_graph([[0, 2**31]])


@pytest.mark.parametrize("name", [n for n in GOLDEN_NAMES if n not in ("nhint_drop_empty",)])
@pytest.mark.parametrize("M", [12, 39])
def test_cpaa_bitexact_mode_is_bitwise_reference(cheb, name, M):
    z = load_golden(name)
    g = cheb.build_graph(z["edges"], cheb.BuildOptions(**build_kw(name))).graph
    r = cheb.run_cpaa(g, cheb.SolverConfig(rounds=M, mode=cheb.MODE_BITEXACT))
    assert np.array_equal(r.ranks, z[f"cpaa{M}_ranks"])
    assert np.array_equal([t.S_k for t in r.trace], z[f"cpaa{M}_S"])
    assert np.array_equal([t.mass_T for t in r.trace], z[f"cpaa{M}_massT"])
    assert r.total_mass == float(z[f"cpaa{M}_total"])


@pytest.mark.parametrize("name", GOLDEN_NAMES)
@pytest.mark.parametrize("M", [12, 39])
def test_cpaa_fast_within_1e12(cheb, name, M):
    z = load_golden(name)
    g = cheb.build_graph(z["edges"], cheb.BuildOptions(**build_kw(name))).graph
    r = cheb.run_cpaa(g, cheb.SolverConfig(rounds=M))
    ref = z[f"cpaa{M}_ranks"]
    assert np.max(np.abs(r.ranks - ref)) <= TOL64
    if g.n >= 200:
        assert np.array_equal(top_k(r.ranks), top_k(ref))
    S = np.array([t.S_k for t in r.trace])
    assert np.all(np.abs(S - z[f"cpaa{M}_S"]) <= g.n * 1e-12)


def test_cpaa_fp32_within_relative_l1(cheb):
    z = load_golden("config1")
    g = cheb.build_graph(z["edges"]).graph
    r = cheb.run_cpaa(g, cheb.SolverConfig(rounds=39, precision=32))
    ref = z["cpaa39_ranks"]
    assert np.sum(np.abs(r.ranks - ref)) / np.sum(np.abs(ref)) <= TOL32_L1


def test_config1_eps_planning_and_top100(cheb):
    z = load_golden("config1")
    dg, info = cheb.build_device_graph(z["edges"])
    r = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    assert r.rounds == 39
    assert np.max(np.abs(r.ranks - z["cpaa39_ranks"])) <= TOL64
    assert np.array_equal(top_k(r.ranks), top_k(z["cpaa39_ranks"]))
    # a resident handle can be re-solved (CUDA-graph replay) with identical bits
    r2 = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    assert np.array_equal(r.ranks, r2.ranks)
    dg.free()


@pytest.mark.parametrize("mode", [0, 1])
def test_power_against_fixture(cheb, mode):
    for name in ("path3", "gnp500", "config1", "star100"):
        z = load_golden(name)
        g = cheb.build_graph(z["edges"]).graph
        p = cheb.run_power(g, cheb.PowerConfig(rounds=210, mode=mode))
        if mode == cheb.MODE_BITEXACT:
            assert np.array_equal(p.ranks, z["power210_ranks"])
            assert np.array_equal([t.l1_change for t in p.trace], z["power210_l1"])
        else:
            assert np.max(np.abs(p.ranks - z["power210_ranks"])) <= TOL64


@pytest.mark.parametrize("mode", [0, 1])
def test_transition_apply(cheb, mode):
    for name in ("path3", "star4", "selfloop", "gnp2000", "config1"):
        z = load_golden(name)
        g = cheb.build_graph(z["edges"]).graph if name != "selfloop" else cheb.build_graph(z["edges"]).graph
        y = cheb.transition_apply(g, z["tapply_x"], mode=mode)
        if mode == cheb.MODE_BITEXACT:
            assert np.array_equal(y, z["tapply_y"])
        else:
            assert np.max(np.abs(y - z["tapply_y"])) <= 1e-12


@pytest.mark.parametrize("mode", [0, 1])
def test_staged_equals_fused_bitwise(cheb, oracle, mode):
    # test_cpaa.cpp:157-173, in both modes
    g = oracle.build_graph(oracle.gnp_edges(500, 0.012, 7))
    G = cheb.UndirectedGraph(g.n, g.m, g.offsets, g.neighbors, g.degrees, g.inv_degree)
    M = 9
    t = cheb.coefficients(C, M)
    st = cheb.init_state(G, t.c0, mode=mode)
    for k in range(1, M + 1):
        cheb.generate_stage(st)
        cheb.accumulate_stage(st, t.coeffs[k])
        st.rotate()
    acc = st.acc
    st.close()
    fused = cheb.run_cpaa(G, cheb.SolverConfig(rounds=M, mode=mode))
    if mode == cheb.MODE_BITEXACT:
        manual = cheb.normalize(acc)
        assert np.array_equal(manual, fused.ranks)
        assert cheb.kahan_sum(acc) == fused.total_mass
    else:
        assert np.max(np.abs(acc / fused.total_mass - fused.ranks)) <= 1e-15


def test_staged_recurrence_examples(cheb):
    # test_cpaa.cpp:105-123
    k2 = cheb.build_graph([[0, 1]]).graph
    t = cheb.coefficients(C, 3)
    st = cheb.init_state(k2, t.c0)
    cheb.generate_stage(st)
    assert st.T_next.tolist() == [1.0, 1.0]
    st.close()
    p3 = cheb.build_graph([[0, 1], [1, 2]]).graph
    st = cheb.init_state(p3, t.c0)
    st.set(T_prev=np.ones(3), T_curr=np.array([0.5, 2.0, 0.5]), k=2)
    cheb.generate_stage(st)
    assert st.T_next.tolist() == [1.0, 1.0, 1.0]
    st.close()
    st = cheb.init_state(k2, t.c0)
    cheb.generate_stage(st)
    cheb.accumulate_stage(st, cheb.coefficients(C, 1).coeffs[1])
    assert abs(st.acc[0] - 4.0120006773991105) <= 1e-12
    st.close()


def test_error_paths(cheb):
    p3 = cheb.build_graph([[0, 1], [1, 2]]).graph
    bad = cheb.UndirectedGraph(p3.n, p3.m, p3.offsets, p3.neighbors, p3.degrees, p3.inv_degree.copy())
    bad.inv_degree[1] = 1e308  # test_cpaa.cpp:371-376
    for mode in (0, 1):
        with pytest.raises(cheb.NumericError, match="round"):
            cheb.run_cpaa(bad, cheb.SolverConfig(rounds=5, mode=mode))
        with pytest.raises(cheb.NumericError, match="round"):
            cheb.run_power(bad, cheb.PowerConfig(rounds=9, mode=mode))
    iso = cheb.UndirectedGraph(2, 0, np.array([0, 0, 0]), np.zeros(0, np.int64), np.array([0, 0]), np.zeros(2))
    with pytest.raises(cheb.ValidationError):
        cheb.run_cpaa(iso, cheb.SolverConfig(rounds=3))
    with pytest.raises(ValueError):
        cheb.run_cpaa(p3, cheb.SolverConfig(rounds=5, eps=1e-3))
    with pytest.raises(ValueError):
        cheb.run_cpaa(p3, cheb.SolverConfig())
    with pytest.raises(ValueError):
        cheb.run_cpaa(p3, cheb.SolverConfig(rounds=5), reference=np.ones(5))
    with pytest.raises(cheb.DomainError):
        cheb.run_cpaa(p3, cheb.SolverConfig(rounds=5, c=1.0))
    with pytest.raises(ValueError):
        cheb.run_power(p3, cheb.PowerConfig(rounds=5, tol=1e-3))
    with pytest.raises(cheb.DomainError):
        cheb.run_power(p3, cheb.PowerConfig(rounds=5, c=1.0))
    with pytest.raises(ValueError):
        cheb.transition_apply(p3, np.ones(5))


def test_rounds_resolution_through_solver(cheb):
    p3 = cheb.build_graph([[0, 1], [1, 2]]).graph
    assert cheb.run_cpaa(p3, cheb.SolverConfig(eps=1e-3)).rounds == 12
    assert cheb.run_cpaa(p3, cheb.SolverConfig(eps=1e-30)).rounds == 60
    r = cheb.run_cpaa(p3, cheb.SolverConfig(rounds=7))
    assert r.rounds == 7 and len(r.trace) == 7
    assert cheb.run_cpaa(p3, cheb.SolverConfig(rounds=90, max_rounds=90)).rounds == 90
    c4 = cheb.build_graph([[0, 1], [1, 2], [2, 3], [3, 0]]).graph
    r0 = cheb.run_cpaa(c4, cheb.SolverConfig(rounds=0))
    assert r0.rounds == 0 and r0.trace == [] and np.allclose(r0.ranks, 0.25, rtol=1e-14)


def test_reference_tracking_columns(cheb):
    z = load_golden("gnp2000")
    g = cheb.build_graph(z["edges"]).graph
    ref = z["power210_ranks"]
    r = cheb.run_cpaa(g, cheb.SolverConfig(rounds=40), reference=ref)
    assert r.has_err
    crossing = next(t.k for t in r.trace if t.err < 1e-3)
    assert 10 <= crossing <= 14  # test_cpaa.cpp:301-329
    plain = cheb.run_cpaa(g, cheb.SolverConfig(rounds=40))
    assert np.array_equal(plain.ranks, r.ranks)
    p = cheb.run_power(g, cheb.PowerConfig(rounds=40), reference=ref)
    assert p.trace[0].err > p.trace[-1].err


def test_chung_lu_and_rmat_against_oracle(cheb, oracle):
    from paper_2112_01743_b200 import generate as G
    cases = [(G.chung_lu_edges(1 << 14, draws=150_000, seed=5), {}),
             (G.rmat_edges(14, 16, seed=3), {"drop_isolated": True})]
    for e, kw in cases:
        e64 = e.astype(np.int64)
        ref = oracle.build_graph(e64, **kw)
        res = cheb.build_graph(e64, cheb.BuildOptions(**kw))
        g = res.graph
        assert np.array_equal(g.offsets, ref.offsets) and np.array_equal(g.neighbors, ref.neighbors)
        assert res.isolated_dropped == ref.isolated_dropped
        assert res.duplicates_removed == ref.duplicates_removed
        o = oracle.run_cpaa(ref, 39)
        fast = cheb.run_cpaa(g, cheb.SolverConfig(rounds=39))
        assert np.max(np.abs(fast.ranks - o.ranks)) <= TOL64
        assert np.array_equal(top_k(fast.ranks), top_k(o.ranks))
        exact = cheb.run_cpaa(g, cheb.SolverConfig(rounds=39, mode=cheb.MODE_BITEXACT))
        assert np.array_equal(exact.ranks, o.ranks)
        f32 = cheb.run_cpaa(g, cheb.SolverConfig(rounds=39, precision=32))
        assert np.sum(np.abs(f32.ranks - o.ranks)) / np.sum(o.ranks) <= TOL32_L1


def test_device_generators_match_host(cheb):
    from paper_2112_01743_b200 import generate as G
    import ctypes as Cc
    for fn, args in [(G.rmat_edges, (13, 16, 0.57, 0.19, 0.19, 11)),
                     (G.chung_lu_edges, (1 << 13, 2.1, 2.0, 500.0, 60_000, 4))]:
        h = fn(*args)
        d = fn(*args, device=0)
        buf = np.zeros(d.count * 2, dtype=np.int32)
        from paper_2112_01743_b200 import _lib
        import ctypes
        cudart = ctypes.CDLL("libcudart.so") if False else None
        # read back through the builder: device edges -> CSR == host edges -> CSR
        dg_info = None
        lib = _lib.load()
        o = _lib.cheb_build_opts(1, 1, 0, 0, 0)
        hnd = Cc.c_void_p()
        inf = _lib.cheb_graph_info()
        rc = lib.cheb_graph_build_device(Cc.c_void_p(d.ptr), d.count, 32, Cc.byref(o), Cc.byref(hnd), Cc.byref(inf))
        assert rc == 0
        dgraph = cheb.DeviceGraph(hnd, inf.n).download()
        hgraph = cheb.build_graph(h.astype(np.int64), cheb.BuildOptions(drop_isolated=True)).graph
        assert d.count == h.shape[0]
        assert np.array_equal(dgraph.offsets, hgraph.offsets)
        assert np.array_equal(dgraph.neighbors, hgraph.neighbors)
        d.free()


@pytest.mark.parametrize("precision", [64, 32])
def test_batched_seeds_against_oracle(cheb, oracle, precision):
    """K5 batched SpMM: each one-hot column equals the oracle run with T0 = e_seed."""
    from paper_2112_01743_b200 import generate as G
    for e, R in [(oracle.gnp_edges(2000, 0.003, 3), 8),
                 (G.chung_lu_edges(1 << 13, draws=60_000, seed=9).astype(np.int64), 64),
                 (oracle.gnp_edges(500, 0.012, 7), 33)]:
        g_or = oracle.build_graph(e)
        g = cheb.build_graph(e).graph
        rng = np.random.default_rng(R)
        seeds = rng.choice(g.n, size=R, replace=False)
        res = cheb.run_cpaa_batch(g, cheb.SolverConfig(rounds=39, precision=precision), seeds=seeds)
        assert res.ranks.shape == (g.n, R)
        for r in range(R):
            p = np.zeros(g.n)
            p[seeds[r]] = 1.0
            want = oracle.run_cpaa(g_or, 39, p=p).ranks
            got = res.ranks[:, r]
            if precision == 64:
                assert np.max(np.abs(got - want)) <= TOL64
            else:
                assert np.sum(np.abs(got - want)) / np.sum(np.abs(want)) <= TOL32_L1


def test_batched_dense_personalization_and_uniform_column(cheb, oracle):
    z = load_golden("gnp2000")
    g = cheb.build_graph(z["edges"]).graph
    g_or = oracle.build_graph(z["edges"])
    rng = np.random.default_rng(1)
    P = rng.random((g.n, 3)) + 0.1
    P[:, 0] = 1.0  # uniform column = the reference's own run
    res = cheb.run_cpaa_batch(g, cheb.SolverConfig(rounds=39), personalization=P)
    assert np.max(np.abs(res.ranks[:, 0] - z["cpaa39_ranks"])) <= TOL64
    for r in (1, 2):
        want = oracle.run_cpaa(g_or, 39, p=P[:, r]).ranks
        assert np.max(np.abs(res.ranks[:, r] - want)) <= TOL64
    # scalar path with an explicit personalisation vector agrees too
    single = cheb.run_cpaa(g, cheb.SolverConfig(rounds=39, personalization=P[:, 1]))
    assert np.max(np.abs(single.ranks - res.ranks[:, 1])) <= TOL64


def test_nccl_partitioned_path_single_rank(cheb):
    """The multi-GPU code path (NCCL communicator attached, per-term all-gather, rank-ordered
    trace combine, slot gather + un-shuffle + un-permute) at world size 1 on one B200: identical bits
    to the single-GPU solve.  Multi-rank correctness is covered on CPU by
    tests/test_multigpu_cpu.py (same plan and exchange protocol)."""
    from paper_2112_01743_b200.distributed import Communicator, partition_info
    for name in ("config1", "gnp2000", "star100"):
        z = load_golden(name)
        dg, _ = cheb.build_device_graph(z["edges"])
        plain = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
        comm = Communicator(0, 1, 0)
        comm.attach(dg)
        info = partition_info(dg)
        assert info["rows"] == int(z["n"]) and info["max_rows"] == int(z["n"])
        part = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
        assert np.array_equal(part.ranks, plain.ranks)
        assert np.max(np.abs(part.ranks - z["cpaa39_ranks"])) <= TOL64
        dg.free()
        comm.close()


def test_int64_row_pointer_solves(cheb):
    """Config 4 uses int64 row pointers: the same solves on an rp64 handle."""
    for name in ("gnp2000", "star100", "config1"):
        z = load_golden(name)
        dg, info = cheb.build_device_graph(z["edges"], cheb.BuildOptions(row_ptr_64=True))
        assert info["row_ptr_64"] == 1
        g = dg.download()
        assert np.array_equal(g.offsets, z["offsets"]) and np.array_equal(g.neighbors, z["neighbors"])
        fast = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
        assert np.max(np.abs(fast.ranks - z["cpaa39_ranks"])) <= TOL64
        exact = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39, mode=cheb.MODE_BITEXACT))
        assert np.array_equal(exact.ranks, z["cpaa39_ranks"])
        p = cheb.run_power(dg, cheb.PowerConfig(rounds=210))
        assert np.max(np.abs(p.ranks - z["power210_ranks"])) <= TOL64
        b = cheb.run_cpaa_batch(dg, cheb.SolverConfig(rounds=39), personalization=np.ones((g.n, 2)))
        assert np.max(np.abs(b.ranks[:, 1] - z["cpaa39_ranks"])) <= TOL64
        dg.free()


def test_pageable_upload_host_narrowing(cheb):
    """Pageable (numpy) CSR arrays of >= 2^22 entries take the host-narrowing path (threads
    narrow int64 -> int32 into a pinned ring while the DMA runs): same device CSR, same
    solve, and the first out-of-range neighbour reported at its exact entry."""
    from paper_2112_01743_b200 import generate as Gen
    e = Gen.chung_lu_edges(1 << 18, 2.1, 2.0, 5000.0, 3_000_000, 21)
    dg, info = cheb.build_device_graph(e)
    assert info["nnz"] >= (1 << 22)
    host = dg.download()
    up = cheb.upload(host)
    back = up.download()
    assert np.array_equal(back.offsets, host.offsets) and np.array_equal(back.neighbors, host.neighbors)
    a = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
    b = cheb.run_cpaa(up, cheb.SolverConfig(rounds=39))
    assert np.array_equal(a.ranks, b.ranks)
    bad = host.neighbors.copy()
    bad[4_500_001] = host.n
    bad[4_600_000] = -3
    g2 = cheb.UndirectedGraph(host.n, host.m, host.offsets, bad, host.degrees, host.inv_degree, host.multi)
    with pytest.raises(cheb.ValidationError, match="out of range at entry 4500001"):
        cheb.upload(g2)
    # host checks split over threads (n >= 2^18): the lowest failing vertex, reference order
    def upload_with(deg=None, off=None):
        g3 = cheb.UndirectedGraph(host.n, host.m, host.offsets if off is None else off, host.neighbors,
                                  host.degrees if deg is None else deg, host.inv_degree, host.multi)
        return cheb.upload(g3)
    deg = host.degrees.copy()
    deg[250_000] = 0
    deg[200_001] = 0
    with pytest.raises(cheb.ValidationError, match=r"vertex 200001 is isolated \(degree 0\)"):
        upload_with(deg=deg)
    deg[10] = 0
    with pytest.raises(cheb.ValidationError, match=r"vertex 10 is isolated"):
        upload_with(deg=deg)
    off = host.offsets.copy()
    off[230_000] = off[230_001] + 1
    off[240_000] = off[240_001] + 1
    with pytest.raises(cheb.ValidationError, match="offsets not monotone at vertex 230000"):
        upload_with(off=off)
    deg = host.degrees.copy()
    deg[255_000] = 0                                   # isolated is checked before monotone
    with pytest.raises(cheb.ValidationError, match="vertex 255000 is isolated"):
        upload_with(deg=deg, off=off)


def test_batched_more_than_one_block(cheb):
    """R = 200 right-hand sides (beyond one 128-column SpMM pass): column blocks give the
    same columns as a single block and as the scalar personalised solves."""
    z = load_golden("gnp2000")
    dg, _ = cheb.build_device_graph(z["edges"])
    rng = np.random.default_rng(3)
    seeds = rng.choice(int(z["n"]), 200, replace=False).astype(np.int64)
    big = cheb.run_cpaa_batch(dg, cheb.SolverConfig(rounds=39), seeds=seeds)
    assert big.ranks.shape == (int(z["n"]), 200)
    small = cheb.run_cpaa_batch(dg, cheb.SolverConfig(rounds=39), seeds=seeds[:128])
    assert np.array_equal(big.ranks[:, :128], small.ranks)
    for r in (0, 127, 128, 199):
        p = np.zeros(int(z["n"]))
        p[seeds[r]] = 1.0
        one = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39, personalization=p))
        assert np.max(np.abs(one.ranks - big.ranks[:, r])) <= 1e-12


def test_device_validate_matches_reference(cheb, reference):
    """cheb_validate_csr (graph.cpp:123-186 on the device) against the reference's own
    validate on randomly corrupted CSRs: the same first error message, or the same stats.
    Corruptions keep every row inside the neighbour array (the reference would read out of
    bounds otherwise)."""
    from oracle import CSR, OracleError
    rng = np.random.default_rng(17)
    checked = 0
    for name in ("config1", "gnp500", "selfloop", "multi", "star100"):
        z = load_golden(name)
        multi = name == "multi"
        base = CSR(int(z["n"]), int(z["m"]), z["offsets"].copy(), z["neighbors"].copy(), z["degrees"].copy(),
                   1.0 / z["degrees"].astype(np.float64), 0, 0, multi)
        for trial in range(40):
            off, nb, deg, m = base.offsets.copy(), base.neighbors.copy(), base.degrees.copy(), base.m
            kind = trial % 6
            i = int(rng.integers(0, nb.size))
            v = int(rng.integers(0, base.n))
            if kind == 0:
                nb[i] = int(rng.integers(-2, base.n + 2))          # range / order / duplicate / symmetry
            elif kind == 1 and nb.size > 1:
                j = int(rng.integers(0, nb.size))
                nb[i], nb[j] = nb[j], nb[i]                         # order / symmetry
            elif kind == 2:
                deg[v] += int(rng.choice([-1, 1]))                  # degree mismatch
            elif kind == 3:
                m += int(rng.choice([-1, 1]))                       # edge count
            elif kind == 4 and 0 < v < base.n:
                off[v] = off[v + 1] + 1 if off[v + 1] + 1 <= nb.size else off[v]   # non-monotone, in bounds
            elif kind == 5 and 0 < v < base.n:
                off[v] = off[v - 1]                                 # empty row -> isolated / degree
            g = CSR(base.n, m, off, nb, deg, base.inv_degree, 0, 0, multi)
            try:
                want = ("ok", reference.graph_from_csr(g).validate())
            except OracleError as e:
                want = ("error", e.msg)
            try:
                st = cheb.validate(cheb.UndirectedGraph(g.n, g.m, off, nb, deg, base.inv_degree, multi))
                got = ("ok", dict(n=st.n, m=st.m, min_degree=st.min_degree, max_degree=st.max_degree,
                                  self_loops=st.self_loops))
            except cheb.ValidationError as e:
                got = ("error", str(e))
            assert got == want, (name, trial, kind, got, want)
            checked += 1
    assert checked == 200


def test_bank_aware_chunk_order_is_a_reassociation(cheb):
    """Hub-row chunks are stored in bank-aware order (k_permute_chunks): the same solve with
    the storage order kept agrees within 1e-12 with identical top-100, and each layout is
    deterministic."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 5000.0, 600_000, 5)
    runs = {}
    try:
        for sched in (1, 0):
            assert lib.cheb_set_tuning(b"chunksched", sched) == 0
            dg, info = cheb.build_device_graph(e)
            a = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
            b = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
            assert np.array_equal(a.ranks, b.ranks)
            runs[sched] = a.ranks
            dg.free()
    finally:
        lib.cheb_set_tuning(b"chunksched", 1)
    assert info["max_degree"] > 248                       # hub rows exist (chunk tiles)
    assert np.max(np.abs(runs[1] - runs[0])) <= TOL64
    top = lambda r: np.argsort(-r, kind="stable")[:100]  # noqa: E731
    assert np.array_equal(top(runs[1]), top(runs[0]))


def _view(lib, dg):
    import ctypes as C
    sizes = np.zeros(5, dtype=np.int64)
    P64 = C.POINTER(C.c_int64)
    assert lib.cheb_graph_view_download(dg.handle, sizes.ctypes.data_as(P64), None, None, None, None) == 0
    nl, nnz, n_hub, nct, H = (int(v) for v in sizes)
    rp = np.zeros(nl + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int32)
    order = np.zeros(nl, dtype=np.int32)
    cb = np.zeros(nct + 1, dtype=np.int64)
    P32 = C.POINTER(C.c_int32)
    assert lib.cheb_graph_view_download(dg.handle, sizes.ctypes.data_as(P64), rp.ctypes.data_as(P64),
                                        col.ctypes.data_as(P32), order.ctypes.data_as(P32),
                                        cb.ctypes.data_as(P64)) == 0
    return dict(rp=rp, col=col, order=order, chunks=cb, n_hub=n_hub, H=H)


def test_bank_aware_chunk_order_permutes_each_chunk(cheb):
    """The bank-aware chunk schedule (k_permute_chunks) is a real per-chunk permutation: each
    hub-row chunk holds the same multiset of ids with and without it, some chunks are
    reordered, and where reordered each half-warp window of 16 positions reads its hot-prefix
    ids (< H) from distinct bank pairs (id mod 16).  Rows, row pointers and the relabel are
    identical."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 5000.0, 600_000, 5)
    views = {}
    try:
        for sched in (1, 0):
            assert lib.cheb_set_tuning(b"chunksched", sched) == 0
            dg, _ = cheb.build_device_graph(e)
            views[sched] = _view(lib, dg)
            dg.free()
    finally:
        lib.cheb_set_tuning(b"chunksched", 1)
    a, b = views[1], views[0]
    assert np.array_equal(a["rp"], b["rp"]) and np.array_equal(a["order"], b["order"])
    assert np.array_equal(a["chunks"], b["chunks"]) and a["chunks"].size > 1
    hub_end = int(a["rp"][a["n_hub"]])
    assert np.array_equal(a["col"][hub_end:], b["col"][hub_end:])  # pack rows untouched
    H = a["H"]
    reordered = 0
    for t in range(a["chunks"].size - 1):
        z0, z1 = int(a["chunks"][t]), int(a["chunks"][t + 1])
        ca, cb = a["col"][z0:z1], b["col"][z0:z1]
        assert np.array_equal(np.sort(ca), np.sort(cb)), t
        if not np.array_equal(ca, cb):
            reordered += 1
            for w0 in range(0, z1 - z0, 16):
                win = ca[w0:w0 + 16]
                hot = win[win < H]
                assert np.unique(hot & 15).size == hot.size, (t, w0)
    assert reordered > 0


@pytest.mark.parametrize("mode", ["fast", "bitexact"])
def test_trace_elapsed_is_per_term_device_time(cheb, mode):
    """TraceRow::elapsed_ms is each term's own device time (%globaltimer stamps at the term
    boundaries inside the solve, graph replay included), not the loop mean: positive,
    finite, and summing to no more than the solve's device loop."""
    import ctypes as C
    from paper_2112_01743_b200 import _lib as L
    z = load_golden("config1")
    dg, _ = cheb.build_device_graph(z["edges"])
    cfg = cheb.SolverConfig(eps=1e-10, mode=cheb.MODE_FAST if mode == "fast" else cheb.MODE_BITEXACT)
    for _ in range(3):  # plain launches, then a captured graph, then a replay
        r = cheb.run_cpaa(dg, cfg)
        el = np.array([t.elapsed_ms for t in r.trace])
        assert el.size == 39 and np.all(np.isfinite(el)) and np.all(el > 0), el
        lm = C.c_double()
        assert L.load().cheb_last_timing(dg.handle, C.byref(lm), None, None, None) == 0
        assert el.sum() <= lm.value * 1.05 + 0.05, (el.sum(), lm.value)
        assert len(set(np.round(el, 9))) > 1  # not one mean repeated
    dg.free()


def _greedy_tiles(deg):
    """The view's greedy tiling restated per row (build.cu make_tile_segs expands the same
    tiles per run on the device): hub rows (degree > 248) in 248-entry chunks, then pack tiles
    of <= 32 consecutive rows and <= 248 entries, lanes per row from the first row's degree."""
    W, RW = 248, 32

    def lanes_log2(dmax, rows):
        lg = 0
        while lg < 5 and (rows << (lg + 1)) <= 32 and (4 << (lg + 1)) <= dmax + 3:
            lg += 1
        return lg

    tiles = []
    z = 0
    cur = None  # [z0, row0, dmax, rows, nnz]
    for r, d in enumerate(deg.tolist()):
        if d > W:
            for j in range(0, d, W):
                tiles.append((z + j, r, 0x10))
            z += d
            continue
        if cur is not None and (cur[3] == RW or (W - cur[4]) < d):
            tiles.append((cur[0], cur[1], lanes_log2(cur[2], cur[3])))
            cur = None
        if cur is None:
            cur = [z, r, d, 0, 0]
        cur[3] += 1
        cur[4] += d
        z += d
        if cur[3] == RW or W - cur[4] < d:
            tiles.append((cur[0], cur[1], lanes_log2(cur[2], cur[3])))
            cur = None
    if cur is not None:
        tiles.append((cur[0], cur[1], lanes_log2(cur[2], cur[3])))
    tiles.append((z, deg.size, 0))
    return tiles


def _tiles(lib, dg):
    import ctypes as C
    nt = C.c_int64()
    nl = C.c_int32()
    assert lib.cheb_graph_view_tiles(dg.handle, C.byref(nt), None, None, None, C.byref(nl)) == 0
    z = np.zeros(nt.value + 1, dtype=np.int64)
    r = np.zeros(nt.value + 1, dtype=np.int32)
    m = np.zeros(nt.value + 1, dtype=np.int32)
    P32 = C.POINTER(C.c_int32)
    assert lib.cheb_graph_view_tiles(dg.handle, C.byref(nt), z.ctypes.data_as(C.POINTER(C.c_int64)),
                                     r.ctypes.data_as(P32), m.ctypes.data_as(P32), C.byref(nl)) == 0
    return z, r, m, nl.value


@pytest.mark.parametrize("graph", ["chung_lu", "rmat", "fixture"])
def test_device_tiling_matches_the_greedy_rule(cheb, graph):
    """The tiles written on the device from per-run segments (k_expand_tiles) are exactly the
    greedy per-row tiling: same first entry, row and lanes per row for every tile."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    if graph == "chung_lu":
        e = Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 5000.0, 600_000, 5)
    elif graph == "rmat":
        e = Gen.rmat_edges(15, 16, 0.57, 0.19, 0.19, 7)
    else:
        e = load_golden("config1")["edges"]
    dg, _ = cheb.build_device_graph(e, cheb.BuildOptions(drop_isolated=graph == "rmat"))
    try:
        v = _view(lib, dg)
        z, r, m, launches = _tiles(lib, dg)
    finally:
        dg.free()
    deg = np.diff(v["rp"])
    assert np.all(deg[:-1] >= deg[1:])  # degree-descending view rows
    ref = _greedy_tiles(deg)
    assert launches == 1
    assert z.size == len(ref)
    assert np.array_equal(z, np.array([t[0] for t in ref], dtype=np.int64))
    assert np.array_equal(r, np.array([t[1] for t in ref], dtype=np.int32))
    assert np.array_equal(m, np.array([t[2] for t in ref], dtype=np.int32))


def test_column_block_schedule_is_a_reassociation(cheb):
    """Opt-in column-blocked schedule (colblocks = K on a view with ascending-id rows): one
    term launch per block of x, no hub-row chunk gathers across a block boundary, every hub
    row's entries still covered once in order, and the ranks stay within the FAST bar of the
    single-launch schedule with the same top-100."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 5000.0, 600_000, 5)
    K = 3
    res = {}
    try:
        assert lib.cheb_set_tuning(b"sortrows", 1) == 0
        for cb in (0, K):
            assert lib.cheb_set_tuning(b"colblocks", cb) == 0
            dg, _ = cheb.build_device_graph(e)
            try:
                v = _view(lib, dg)
                z, r, m, launches = _tiles(lib, dg)
                res[cb] = (cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks, v, z, r, m, launches)
            finally:
                dg.free()
    finally:
        lib.cheb_set_tuning(b"colblocks", 0)
        lib.cheb_set_tuning(b"sortrows", -1)
    ranks0, v0, *_ = res[0]
    ranks, v, z, r, m, launches = res[K]
    assert launches == K
    assert np.array_equal(v["rp"], v0["rp"]) and np.array_equal(v["col"], v0["col"])
    n = v["rp"].size - 1
    bounds = [0] + [(n * j // K) & ~31 for j in range(1, K)] + [n]
    col = v["col"]
    chunk = (m & 0x10) != 0
    assert chunk.any()
    for t in np.nonzero(chunk)[0]:
        ids = col[z[t]:z[t + 1]]
        assert ids.size <= 248
        blk = np.searchsorted(bounds, ids, side="right") - 1
        assert np.all(blk == blk[0]), t
    # chunk tiles of a hub row tile its entries contiguously, in order
    hub_rows = np.unique(r[chunk])
    n_hub = int(hub_rows.size)
    assert np.array_equal(hub_rows, np.arange(n_hub))
    first = np.nonzero(chunk)[0]
    assert z[first[0]] == 0 and z[first[-1] + 1] == v["rp"][n_hub]
    assert np.max(np.abs(ranks - ranks0)) <= TOL64
    top = lambda x: np.argsort(-x, kind="stable")[:100]  # noqa: E731
    assert np.array_equal(top(ranks), top(ranks0))


@pytest.mark.parametrize("precision", [64, 32])
def test_hub_finalize_lane_rows_bitwise_equal_warp_rows(cheb, precision):
    """Hub rows with <= 32 chunk partials are finalized by one lane replaying the warp's
    shuffle-tree sum: ranks and trace bitwise equal to finalizing every hub row with a warp."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = Gen.chung_lu_edges(1 << 17, 2.1, 2.0, 20000.0, 2_000_000, 9)
    dg, info = cheb.build_device_graph(e)
    out = {}
    try:
        for hw in (0, 1):
            assert lib.cheb_set_tuning(b"hubwarp", hw) == 0
            out[hw] = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, precision=precision))
    finally:
        lib.cheb_set_tuning(b"hubwarp", 0)
        dg.free()
    assert info["max_degree"] > 32 * 248  # both finalize paths run
    assert np.array_equal(out[0].ranks, out[1].ranks)
    assert [t.S_k for t in out[0].trace] == [t.S_k for t in out[1].trace]


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("graph", ["chung_lu", "rmat", "star100"])
def test_single_column_buffer_kernel_bitwise_equal(cheb, graph, precision):
    """The term kernel with one column-id buffer per warp (picked when x exceeds L2) reads each
    tile's ids into registers before refilling the buffer, lanes with more than 8 entries of a
    mixed-degree pack tile included: ranks and trace bitwise equal to the two-buffer kernel."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    if graph == "chung_lu":
        e, kw = Gen.chung_lu_edges(1 << 17, 2.1, 2.0, 20000.0, 2_000_000, 9), {}
    elif graph == "rmat":
        e, kw = Gen.rmat_edges(16, 16, 0.57, 0.19, 0.19, 5), {"drop_isolated": True}
    else:  # the hub (degree 99) shares a pack tile with 31 leaves: one lane walks 99 entries
        e, kw = load_golden("star100")["edges"], {}
    dg, _ = cheb.build_device_graph(e, cheb.BuildOptions(**kw))
    out = {}
    try:
        for nb in (2, 1):
            assert lib.cheb_set_tuning(b"colbufs", nb) == 0
            out[nb] = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, precision=precision))
    finally:
        lib.cheb_set_tuning(b"colbufs", -1)
        dg.free()
    assert np.array_equal(out[1].ranks, out[2].ranks)
    assert [t.S_k for t in out[1].trace] == [t.S_k for t in out[2].trace]


def test_single_column_buffer_kernel_deterministic_at_scale(cheb):
    """One column-id buffer per warp on a graph of ~30 M entries (forced; the product picks it
    when x exceeds L2): repeated solves are bitwise equal to each other and to the two-buffer
    kernel (a refill racing the id reads shows up here as run-to-run differences)."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = Gen.rmat_edges(20, 16, 0.57, 0.19, 0.19, 13)
    dg, info = cheb.build_device_graph(e, cheb.BuildOptions(drop_isolated=True))
    assert info["nnz"] > 20_000_000
    runs = {}
    try:
        for nb in (2, 1, 1, 1):
            assert lib.cheb_set_tuning(b"colbufs", nb) == 0
            runs.setdefault(nb, []).append(cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks)
    finally:
        lib.cheb_set_tuning(b"colbufs", -1)
        dg.free()
    for r in runs[1]:
        assert np.array_equal(r, runs[2][0])


# ---------------- column windows of the hub rows (SolverView::Windows) ----------------

def _window_plan(lib, dg):
    import ctypes as C
    P64, P32, P16 = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_uint16)
    sizes = np.zeros(8, dtype=np.int64)
    assert lib.cheb_graph_view_windows(dg.handle, sizes.ctypes.data_as(P64), None, None, None, None, None) == 0
    NW, W, H0, nb, entries, pieces, MC, listed = (int(v) for v in sizes)
    v = _view(lib, dg)
    wcol = np.zeros(nb * 256, dtype=np.uint16)
    meta = np.zeros(nb * 32, dtype=np.uint16)
    bbase = np.zeros(nb + 1, dtype=np.int32)
    kf = np.zeros(v["n_hub"] + 1, dtype=np.int32)
    klist = np.zeros(max(listed, 1), dtype=np.int32)
    if NW:
        assert lib.cheb_graph_view_windows(dg.handle, sizes.ctypes.data_as(P64), wcol.ctypes.data_as(P16),
                                           meta.ctypes.data_as(P16), bbase.ctypes.data_as(P32),
                                           kf.ctypes.data_as(P32), klist.ctypes.data_as(P32)) == 0
    return dict(NW=NW, W=W, H0=H0, blocks=nb, entries=entries, pieces=pieces, MC=MC, listed=listed, wcol=wcol,
                meta=meta, bbase=bbase, kf=kf, klist=klist[:listed], view=v)


def _forced_windows(lib, nw, size):
    assert lib.cheb_set_tuning(b"windows", nw) == 0
    assert lib.cheb_set_tuning(b"winsize", size) == 0


def _default_windows(lib):
    lib.cheb_set_tuning(b"windows", -1)
    lib.cheb_set_tuning(b"winsize", 28672)


def _check_window_structure(p):
    """The stream of a window plan holds, piece by piece, exactly the hub rows' entries with ids
    in [H0, H0 + NW W): see test_column_windows_hold_every_windowed_entry_once."""
    v = p["view"]
    NW, W, H0, n_hub = p["NW"], p["W"], p["H0"], v["n_hub"]
    rp, col = v["rp"], v["col"]
    hub_end = int(rp[n_hub])
    row_of = np.repeat(np.arange(n_hub), np.diff(rp[:n_hub + 1]))
    c = col[:hub_end].astype(np.int64)
    inw = (c >= H0) & (c < H0 + NW * W)
    assert p["entries"] == int(inw.sum()) > 0
    want = np.sort(row_of[inw] * (1 << 32) + c[inw])
    # stream: start bits -> piece of every position; windows start at block boundaries
    m = p["meta"]
    bits = ((m[:, None] & 0xff) >> np.arange(8)[None, :]) & 1
    starts = bits.reshape(-1).astype(np.int64)
    assert np.all(starts[::256] == 1)                       # a block's first entry starts a piece
    piece_of = np.cumsum(starts) - 1
    assert p["pieces"] == int(starts.sum()) == int(p["bbase"][-1])
    assert np.array_equal(p["bbase"][:-1], piece_of[::256])
    before = (m >> 8).astype(np.int64)                      # pieces started in the block's earlier lanes
    lane_first = np.cumsum(starts.reshape(-1, 8).sum(1).reshape(-1, 32), axis=1)
    assert np.array_equal(before.reshape(-1, 32)[:, 1:], lane_first[:, :-1]) and np.all(before.reshape(-1, 32)[:, 0] == 0)
    wlen = np.bincount(((c[inw] - H0) // W).astype(np.int64), minlength=NW)
    wblocks = (wlen + 255) // 256
    assert p["blocks"] == int(wblocks.sum())
    win_of_block = np.repeat(np.arange(NW), wblocks)
    ids = H0 + np.repeat(win_of_block, 256) * W + p["wcol"].astype(np.int64)
    piece_row = np.full(p["pieces"], -1, dtype=np.int64)
    piece_row[p["klist"]] = np.repeat(np.arange(n_hub), np.diff(p["kf"]))
    assert np.unique(p["klist"]).size == p["listed"]          # a piece belongs to one row
    r = piece_row[piece_of]
    got = np.sort(r[r >= 0] * (1 << 32) + ids[r >= 0])
    assert np.array_equal(got, want)
    assert int((r < 0).sum()) == int(p["blocks"] * 256 - p["entries"])  # the padding only


@pytest.mark.parametrize("graph", ["chung_lu", "rmat"])
def test_column_windows_hold_every_windowed_entry_once(cheb, graph):
    """The window stream of a view (forced: 6 windows of 2048 ids on a small graph) holds, piece by
    piece, exactly the hub rows' entries with ids in [H0, H0 + NW W): every hub row's listed pieces
    give back the multiset of its windowed ids, pieces never cross a 256-entry block, the per-lane
    piece counts and block bases agree with the start bits, and the padding belongs to no row."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = (Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 20000.0, 900_000, 5) if graph == "chung_lu"
         else Gen.rmat_edges(16, 16, 0.57, 0.19, 0.19, 3))
    try:
        _forced_windows(lib, 6, 2048)
        dg, info = cheb.build_device_graph(e, cheb.BuildOptions(drop_isolated=True))
        p = _window_plan(lib, dg)
        dg.free()
    finally:
        _default_windows(lib)
    assert p["NW"] == 6 and p["W"] == 2048 and p["view"]["n_hub"] > 0
    _check_window_structure(p)


@pytest.mark.parametrize("nw,size,h0", [(1, 256, 0), (3, 65536, 0), (500, 256, 0), (500, 1024, -1), (2, 28672, -1),
                                        (64, 8192, 0)])
def test_column_windows_shapes(cheb, nw, size, h0):
    """Window shapes at the edges: one 256-id window, a requested size above what an fp64 window
    may take of shared memory (clamped to 28,928 ids), windows past the end of x (the count is clamped; every hub-row id windowed, no
    chunk tile left), windows from the hot-prefix capacity instead of id 0.  Structure as above,
    ranks equal to the plain schedule within 1e-12 with the same top-100, solves repeatable."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 20000.0, 900_000, 5)
    try:
        _forced_windows(lib, 0, 28672)
        dg, _ = cheb.build_device_graph(e)
        plain = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks
        dg.free()
        _forced_windows(lib, nw, size)
        assert lib.cheb_set_tuning(b"winh0", h0) == 0
        dg, info = cheb.build_device_graph(e)
        p = _window_plan(lib, dg)
        a = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks
        b = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks
        f32 = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, precision=32)).ranks
        dg.free()
    finally:
        _default_windows(lib)
        lib.cheb_set_tuning(b"winh0", 0)
    H0 = 0 if h0 == 0 else p["view"]["H"]
    size = min(size, 28928)
    assert p["H0"] == H0 and p["W"] == size
    assert p["NW"] == min(nw, -(-(info["n"] - H0) // size))     # clamped to the ids there are
    _check_window_structure(p)
    if nw == 500:  # the windows reach the end of x: only ids below H0 are left to the term kernel
        c = p["view"]["col"][:int(p["view"]["rp"][p["view"]["n_hub"]])]
        assert p["entries"] == int((c >= H0).sum())
    assert np.array_equal(a, b)
    assert np.max(np.abs(a - plain)) <= TOL64
    assert np.array_equal(top_k(a), top_k(plain))
    assert np.sum(np.abs(f32 - plain)) / np.sum(plain) <= TOL32_L1


@pytest.mark.parametrize("graph", ["chung_lu", "rmat"])
def test_column_windows_against_reference(cheb, oracle, graph):
    """Solves with the hub rows' column windows (forced on a small graph) against the oracle and
    against the plain schedule: FAST fp64 <= 1e-12 with the same top-100, fp32 <= 1e-6 relative
    L1, Power and transition_apply <= 1e-12, repeated solves bitwise equal, int64 row pointers."""
    from paper_2112_01743_b200 import _lib
    from paper_2112_01743_b200 import generate as Gen
    lib = _lib.load()
    e = (Gen.chung_lu_edges(1 << 16, 2.1, 2.0, 20000.0, 900_000, 5) if graph == "chung_lu"
         else Gen.rmat_edges(16, 16, 0.57, 0.19, 0.19, 3)).astype(np.int64)
    ref = oracle.build_graph(e, drop_isolated=True)
    want = oracle.run_cpaa(ref, 39).ranks
    x = np.random.default_rng(7).random(ref.n)
    res = {}
    try:
        for nw, rp64 in ((0, False), (6, False), (6, True)):
            _forced_windows(lib, nw, 2048)
            dg, info = cheb.build_device_graph(e, cheb.BuildOptions(drop_isolated=True, row_ptr_64=rp64))
            p = _window_plan(lib, dg)
            assert p["NW"] == nw
            a = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
            b = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39))
            assert np.array_equal(a.ranks, b.ranks)
            f32 = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39, precision=32))
            pw = cheb.run_power(dg, cheb.PowerConfig(rounds=60))
            y = cheb.transition_apply(dg, x)
            exact = cheb.run_cpaa(dg, cheb.SolverConfig(rounds=39, mode=cheb.MODE_BITEXACT))
            res[(nw, rp64)] = (a.ranks, f32.ranks, pw.ranks, y)
            assert np.array_equal(exact.ranks, want)
            dg.free()
    finally:
        _default_windows(lib)
    plain = res[(0, False)]
    for key in ((6, False), (6, True)):
        fast, f32, pw, y = res[key]
        assert np.max(np.abs(fast - want)) <= TOL64
        assert np.array_equal(top_k(fast), top_k(want))
        assert np.sum(np.abs(f32 - want)) / np.sum(want) <= TOL32_L1
        assert np.max(np.abs(fast - plain[0])) <= TOL64
        assert np.max(np.abs(pw - plain[2])) <= TOL64
        assert np.max(np.abs(y - plain[3])) <= 1e-12
    assert np.array_equal(res[(6, False)][0], res[(6, True)][0])   # same schedule, wider row pointers

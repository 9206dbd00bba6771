"""The oracle (oracle/cpaa_oracle.c) pinned against the reference's own golden vectors
 and against the reference compiled unmodified (oracle/_ref, committed
fixtures in tests/golden/ made from it).  CPU only."""
import numpy as np
import pytest

from conftest import GOLDEN_NAMES, load_golden

C = 0.85


def test_frozen_coefficients(oracle):
    # /root/reference/proj/tests/test_coefficients.cpp:15-22 (40-digit table)
    frozen = [(0.50, 0.26794919243112271, 2.3094010767585031, 0.61880215351700612, 0.0031897865781070092),
              (0.85, 0.5567262498321918, 3.7966319830099957, 2.1136846858941127, 0.20305187144012912),
              (0.99, 0.86760872747812232, 14.177624100166712, 12.3006304042088, 6.9698433557705565)]
    for c, b, c0, c1, c5 in frozen:
        co, beta, cc0 = oracle.coefficients(c, 60)
        assert abs(beta - b) <= 1e-13 * b
        assert abs(cc0 - c0) <= 1e-13 * c0
        assert abs(co[1] - c1) <= 1e-13 * c1
        assert abs(co[5] - c5) <= 1e-13 * c5


def test_plan_iterations_known_answers(oracle):
    # test_coefficients.cpp:131-136, :105
    assert [oracle.plan_iterations(C, e)[0] for e in (1e-3, 1e-4, 1e-5, 1e-10)] == [12, 16, 20, 39]
    assert oracle.plan_iterations(C, 0.99)[0] == 0
    assert abs(oracle.err_bound(C, 20) - 5.8518532208583129e-06) <= 1e-12 * 5.85e-6


def test_csr_known_answers(oracle):
    # test_graph.cpp:16-81
    g = oracle.build_graph([[0, 1], [1, 2]])
    assert g.offsets.tolist() == [0, 1, 3, 4] and g.neighbors.tolist() == [1, 0, 2, 1]
    g = oracle.build_graph([[0, 1], [1, 0]])
    assert g.m == 1 and g.duplicates_removed == 1
    g = oracle.build_graph([[0, 1], [1, 0], [0, 1]], dedup=False)
    assert g.m == 3 and g.degrees.tolist() == [3, 3]
    g = oracle.build_graph([[0, 1], [0, 0]])
    assert g.degrees.tolist() == [2, 1] and g.neighbors.tolist() == [0, 1, 0]
    g = oracle.build_graph([[0, 1], [3, 4]], drop_isolated=True)
    assert g.n == 4 and g.isolated_dropped == 1 and g.neighbors.tolist() == [1, 0, 3, 2]
    with pytest.raises(Exception, match="vertex 2"):
        oracle.build_graph([[0, 1], [3, 4]])
    with pytest.raises(Exception, match="negative"):
        oracle.build_graph([[0, -1]])


def test_cpaa_known_answers(oracle):
    # test_cpaa.cpp:38-56, :139-155, :87-92
    k2 = oracle.build_graph([[0, 1]])
    r = oracle.run_cpaa(k2, 12)
    assert np.all(np.abs(r.ranks - 0.5) <= 1e-12)
    co, b, c0 = oracle.coefficients(C, 1)
    r1 = oracle.run_cpaa(k2, 1)
    acc0 = r1.total_mass * r1.ranks[0]
    assert abs(acc0 - 4.0120006773991105) <= 1e-12
    p3 = oracle.build_graph([[0, 1], [1, 2]])
    r = oracle.run_cpaa(p3, 40)
    assert abs(r.ranks[0] - 0.25675675675675674) <= 1e-6
    assert abs(r.ranks[1] - 0.48648648648648651) <= 1e-6
    c4 = oracle.build_graph([[0, 1], [1, 2], [2, 3], [3, 0]])
    r0 = oracle.run_cpaa(c4, 0)
    assert np.allclose(r0.ranks, 0.25, rtol=1e-14)


def test_power_known_answers(oracle):
    # test_power.cpp:37-46
    p3 = oracle.build_graph([[0, 1], [1, 2]])
    r = oracle.run_power(p3, rounds=210)
    assert abs(r.ranks[0] - 0.25675675675675674) <= 1e-9
    assert abs(r.ranks[1] - 0.48648648648648651) <= 1e-9


def test_mass_ledger(oracle):
    # test_cpaa.cpp:260-276: S_k = n (c0/2 + sum c_i) within n 1e-12
    g = oracle.build_graph(oracle.gnp_edges(2000, 0.003, 3))
    r = oracle.run_cpaa(g, 60)
    co, b, c0 = oracle.coefficients(C, 60)
    partial = c0 / 2
    for k in range(1, 61):
        partial += co[k]
        assert abs(r.trace[k - 1, 2] - g.n * partial) <= g.n * 1e-12
        assert abs(r.trace[k - 1, 6] - g.n) <= g.n * 1e-12


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_oracle_matches_reference_fixture(oracle, name):
    """Bit-exact: CSR, CPAA ranks + trace, Power ranks, transition_apply."""
    z = load_golden(name)
    kw = {}
    if name == "multi":
        kw["dedup"] = False
    if name in ("drop", "nhint_drop"):
        kw["drop_isolated"] = True
    if name == "nhint_drop":
        kw["n_hint"] = 6
    g = oracle.build_graph(z["edges"], **kw)
    assert g.n == int(z["n"]) and g.m == int(z["m"])
    assert np.array_equal(g.offsets, z["offsets"])
    assert np.array_equal(g.neighbors, z["neighbors"])
    assert np.array_equal(g.degrees, z["degrees"])
    assert g.duplicates_removed == int(z["duplicates_removed"])
    assert g.isolated_dropped == int(z["isolated_dropped"])
    for M in (12, 39):
        r = oracle.run_cpaa(g, M)
        assert np.array_equal(r.ranks, z[f"cpaa{M}_ranks"])
        assert np.array_equal(r.trace[:, 2], z[f"cpaa{M}_S"])
        assert np.array_equal(r.trace[:, 6], z[f"cpaa{M}_massT"])
        assert r.total_mass == float(z[f"cpaa{M}_total"])
    p = oracle.run_power(g, rounds=210)
    assert np.array_equal(p.ranks, z["power210_ranks"])
    assert np.array_equal(p.trace[:, 4], z["power210_l1"])
    assert np.array_equal(oracle.transition_apply(g, z["tapply_x"]), z["tapply_y"])


def test_oracle_vs_live_reference(oracle, reference):
    """Where the reference build is present: random graphs, several K, bit-exact."""
    for n, p, seed in [(300, 0.02, 1), (1500, 0.004, 8), (4000, 0.002, 5)]:
        e = oracle.gnp_edges(n, p, seed)
        assert np.array_equal(e, reference.gnp_edges(n, p, seed))
        g = oracle.build_graph(e)
        rg = reference.build_graph(e)
        for M in (0, 1, 7, 39, 60):
            a = oracle.run_cpaa(g, M)
            for K in (1, 3):
                b = rg.run_cpaa(rounds=M, parallelism=K)
                assert np.array_equal(a.ranks, b.ranks)
        for K in (1, 2, 5):
            assert np.array_equal(oracle.partition_vertices(g, K), rg.partition_vertices(K))


@pytest.mark.parametrize("kind,args", [
    ("rmat", (10, 16, 0.57, 0.19, 0.19, 3)),
    ("rmat", (17, 16, 0.57, 0.19, 0.19, 4)),
    ("rmat", (14, 8, 0.45, 0.15, 0.15, 11)),
    ("chung_lu", (1000, 2.1, 2.0, 50000.0, 5000, 2)),
    ("chung_lu", (1 << 17, 2.1, 2.0, 50000.0, 1_300_000, 5)),
    ("chung_lu", (5000, 2.5, 1.0, 100.0, 3000, 9)),  # sparse: many rewired vertices
])
def test_config_generators_match_product(oracle, kind, args):
    """oracle/synth_gen.c restates the product's counter-based config generators: the same
    edge list, pair for pair and in the same order, as the product's host path (the device
    path is pinned to the host path and to the reference CSR by the GPU tests).  This is
    what lets the CPU legs build the bench graphs without the product library."""
    from paper_2112_01743_b200 import generate as G
    if kind == "rmat":
        mine, prod = oracle.rmat_edges(*args), G.rmat_edges(*args)
    else:
        mine, prod = oracle.chung_lu_edges(*args), G.chung_lu_edges(*args)
    assert mine.dtype == np.int64 and mine.shape == prod.shape
    assert np.array_equal(mine, prod.astype(np.int64))
    assert not np.any(mine[:, 0] == mine[:, 1])  # self-loops dropped

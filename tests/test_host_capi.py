"""Host side of the C-ABI (no GPU needed): the library loads and exports every symbol
include/*.h declares; the coefficient kit, round resolution, partitioning, Kahan sum
and the generators are bit-identical to the oracle / reference."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "chebpr_cuda.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cheb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2112_01743_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding types every one of them
    assert set(syms) <= set(_lib.EXPORTED), set(syms) - set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2112_01743_b200", "lib", "libchebpr_b200.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_coefficients_bit_identical(cheb, oracle):
    for c in (0.3, 0.5, 0.85, 0.95, 0.99):
        t = cheb.coefficients(c, 60)
        co, b, c0 = oracle.coefficients(c, 60)
        assert np.array_equal(t.coeffs, co) and t.beta == b and t.c0 == c0
        for M in (0, 1, 20, 39):
            assert cheb.err_bound(c, M) == oracle.err_bound(c, M)
        for eps in (1e-2, 1e-4, 1e-8, 1e-10, 1e-12):
            p = cheb.plan_iterations(c, eps)
            assert (p.M, p.predicted_err) == oracle.plan_iterations(c, eps)
    assert abs(cheb.sigma(0.85) - 0.5567) <= 5e-5
    for i in range(1, 20):
        assert abs(cheb.sigma(0.05 * i) - cheb.beta(0.05 * i)) <= 1e-12


def test_coefficient_domain_errors(cheb):
    for bad in (0.0, 1.0, -0.3, 1.7):
        with pytest.raises(cheb.DomainError):
            cheb.beta(bad)
    with pytest.raises(cheb.DomainError):
        cheb.coefficients(0.85, -1)
    with pytest.raises(cheb.DomainError):
        cheb.plan_iterations(0.85, 1.0)
    with pytest.raises(cheb.DomainError):
        cheb.err_bound(0.85, -1)


def test_resolve_rounds_semantics(cheb):
    from paper_2112_01743_b200 import _lib
    lib = _lib.load()
    M = C.c_int()
    assert lib.cheb_resolve_rounds(0.85, -1, 1e-3, 60, C.byref(M)) == 0 and M.value == 12
    assert lib.cheb_resolve_rounds(0.85, -1, 1e-30, 60, C.byref(M)) == 0 and M.value == 60
    assert lib.cheb_resolve_rounds(0.85, 90, -1, 60, C.byref(M)) == 0 and M.value == 60
    assert lib.cheb_resolve_rounds(0.85, 90, -1, 90, C.byref(M)) == 0 and M.value == 90
    assert lib.cheb_resolve_rounds(0.85, 5, 1e-3, 60, C.byref(M)) == 4  # both set
    assert lib.cheb_resolve_rounds(0.85, -1, -1, 60, C.byref(M)) == 4   # neither
    assert lib.cheb_resolve_rounds(0.85, 5, -1, -1, C.byref(M)) == 4    # max_rounds < 0


def test_partition_vertices_matches_oracle(cheb, oracle):
    for n, p, s in [(333, 0.03, 2), (2000, 0.003, 11)]:
        g = oracle.build_graph(oracle.gnp_edges(n, p, s))
        G = cheb.UndirectedGraph(g.n, g.m, g.offsets, g.neighbors, g.degrees, g.inv_degree)
        for K in (1, 2, 3, 7, 8):
            cuts = oracle.partition_vertices(g, K)
            got = cheb.partition_vertices(G, K)
            assert [r.begin for r in got] + [got[-1].end] == cuts.tolist()
    with pytest.raises(cheb.DomainError):
        cheb.partition_vertices(G, 0)
    star = oracle.build_graph([[0, 1], [0, 2], [0, 3]])
    S = cheb.UndirectedGraph(star.n, star.m, star.offsets, star.neighbors, star.degrees, star.inv_degree)
    r = cheb.partition_vertices(S, 2)
    assert (r[0].begin, r[0].end, r[1].end) == (0, 1, 4)


def test_kahan_and_normalize(cheb, oracle):
    x = np.full(1_000_000, 0.1)
    assert cheb.kahan_sum(x) == oracle.kahan_sum(x)
    rng = np.random.default_rng(4)
    w = rng.random(50) + 0.01
    assert np.array_equal(cheb.normalize(w), w / oracle.kahan_sum(w))
    assert cheb.normalize([1.0, 3.0]).tolist() == [0.25, 0.75]
    for bad in (np.zeros(3), np.array([1.0, np.nan, 1.0]), -np.ones(3)):
        with pytest.raises(cheb.NumericError):
            cheb.normalize(bad)


def test_reference_generators_bit_identical(oracle, reference):
    from paper_2112_01743_b200 import generate as G
    for args in [(10000, 0.001, 1), (1000, 0.006, 42), (100, 0.001, 3), (50, 0.0, 9), (20, 1.0, 1)]:
        assert np.array_equal(G.gnp_edges(*args), reference.gnp_edges(*args))
    assert np.array_equal(G.ring_edges(4), reference.ring_edges(4))
    assert np.array_equal(G.ring_edges(2), reference.ring_edges(2))
    assert np.array_equal(G.star_edges(5), reference.star_edges(5))
    assert np.array_equal(G.regular_edges(100, 6), reference.regular_edges(100, 6))
    assert np.array_equal(G.regular_edges(6, 3), reference.regular_edges(6, 3))


def test_config_generators_deterministic():
    from paper_2112_01743_b200 import generate as G
    a = G.rmat_edges(12, 16, seed=7)
    b = G.rmat_edges(12, 16, seed=7)
    assert np.array_equal(a, b) and a.dtype == np.int32
    assert not np.any(a[:, 0] == a[:, 1])
    assert a.max() < 4096 and a.min() >= 0
    c = G.chung_lu_edges(1 << 12, draws=40_000, seed=3)
    assert np.array_equal(c, G.chung_lu_edges(1 << 12, draws=40_000, seed=3))
    assert not np.any(c[:, 0] == c[:, 1])
    deg = np.bincount(c.ravel(), minlength=1 << 12)
    assert deg.min() >= 1  # isolated vertices rewired: n is kept


@pytest.mark.gpu
def test_validate_rejects_corruption(cheb, oracle):
    # test_graph.cpp:135-165 (validate runs on the device: cheb_validate_csr)
    g = oracle.build_graph([[0, 1], [1, 2]])
    G = cheb.UndirectedGraph(g.n, g.m, g.offsets, g.neighbors, g.degrees, g.inv_degree)
    st = cheb.validate(G)
    assert (st.n, st.m, st.min_degree, st.max_degree, st.self_loops) == (3, 2, 1, 2, 0)
    import copy
    for mutate in [lambda h: setattr(h, "neighbors", np.array([1, 2, 0, 1])),
                   lambda h: h.neighbors.__setitem__(0, 2),
                   lambda h: h.degrees.__setitem__(1, 1),
                   lambda h: h.neighbors.__setitem__(3, 9),
                   lambda h: setattr(h, "m", 7)]:
        bad = copy.deepcopy(G)
        mutate(bad)
        with pytest.raises(cheb.ValidationError):
            cheb.validate(bad)
    lonely = cheb.UndirectedGraph(1, 0, np.array([0, 0]), np.zeros(0, np.int64), np.array([0]), np.array([0.0]))
    with pytest.raises(cheb.ValidationError):
        cheb.validate(lonely)
    sl = oracle.build_graph([[0, 1], [0, 0]])
    assert cheb.validate(cheb.UndirectedGraph(sl.n, sl.m, sl.offsets, sl.neighbors, sl.degrees, sl.inv_degree)).self_loops == 1

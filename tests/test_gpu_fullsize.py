"""Full-size parity against the REFERENCE ITSELF on the BASELINE.json bench graphs
(configs 2-5, the exact graphs bench.py times).

The reference side never touches the product library: its edge lists come from the
plain-C restatement of the config generators (oracle/synth_gen.c, pinned equal to the
product's generators by tests/test_oracle.py), its CSR from the reference's own
build_graph and its ranks from the reference's own run_cpaa (oracle/_ref = the unmodified
sources, all host threads).  The product side generates on the device and builds with K1.

Checked per config (SURVEY.md §8(c)/(d) bars, north_star):
  * CSR: offsets, neighbours and degrees bit-exact against the reference build_graph, and
    the same m / duplicates_removed / isolated_dropped;
  * FAST fp64 ranks (the product path): max-abs <= 1e-12 and the same top-100 vertices in
    the same order (ties by vertex id);
  * BITEXACT fp64 ranks: bitwise equal, and the S_k / mass_T trace bitwise equal;
  * fp32: relative L1 <= 1e-6;
  * Power (C2, C3; 50 rounds) against the reference's run_power: FAST within 1e-12, BITEXACT
    bitwise, the L1-change trace too; transition_apply (C2, C3) against the reference's;
  * config 5 (batched, 64 one-hot columns): 4 sampled columns against the restated loop
    (oracle/cpaa_oracle.c with T0 = e_seed; the reference has no personalisation), the same
    bars (fp64 1e-12 + top-100, fp32 1e-6), every column a distribution.
"""
import gc

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
C = 0.85
EPS = 1e-10


def top100(r):
    ids = np.arange(r.size)
    return np.lexsort((ids, -r))[:100]


def _reference_side(reference, name):
    """Edges by oracle/synth_gen.c, CSR by the reference's build_graph."""
    import bench
    cfg = bench.CONFIGS[name]
    e = bench.make_edges_host(cfg)
    rg = reference.build_graph(e, dedup=True, drop_isolated=cfg.get("drop", False))
    del e
    gc.collect()
    return rg


def _device_side(name):
    import bench
    return bench.build_device(bench.CONFIGS[name], 0)


def _windows(dg):
    """(windows, windowed entries) of the resident view: the hub rows' column windows
    (k_window_pass) are part of the default schedule from 48 M entries up."""
    import ctypes as C
    from paper_2112_01743_b200 import _lib
    sizes = np.zeros(8, dtype=np.int64)
    assert _lib.load().cheb_graph_view_windows(dg.handle, sizes.ctypes.data_as(C.POINTER(C.c_int64)),
                                               None, None, None, None, None) == 0
    return int(sizes[0]), int(sizes[4])


def _check_csr(rg, dg, info):
    ref = rg.csr()
    assert info["n"] == rg.n and info["m"] == rg.m and info["nnz"] == rg.nnz
    assert info["duplicates_removed"] == rg.duplicates_removed
    assert info["isolated_dropped"] == rg.isolated_dropped
    mine = dg.download()
    assert np.array_equal(mine.offsets, ref.offsets)
    assert np.array_equal(mine.degrees, ref.degrees)
    # neighbours in 256 M-entry slices (C4 holds 1.05 G of them)
    step = 1 << 28
    for a in range(0, ref.neighbors.size, step):
        assert np.array_equal(mine.neighbors[a:a + step], ref.neighbors[a:a + step]), a
    del mine
    gc.collect()


def _check_solves(cheb, rg, dg, threads, fp32=True, bitexact=True):
    want = rg.run_cpaa(c=C, eps=EPS, parallelism=threads)
    assert want.rounds == 39
    fast = cheb.run_cpaa(dg, cheb.SolverConfig(c=C, eps=EPS))
    assert fast.rounds == 39
    err = float(np.max(np.abs(fast.ranks - want.ranks)))
    assert err <= 1e-12, err
    assert np.array_equal(top100(fast.ranks), top100(want.ranks))
    if bitexact:
        exact = cheb.run_cpaa(dg, cheb.SolverConfig(c=C, eps=EPS, mode=cheb.MODE_BITEXACT))
        assert np.array_equal(exact.ranks, want.ranks)
        s_k = np.array([r.S_k for r in exact.trace])
        m_t = np.array([r.mass_T for r in exact.trace])
        assert np.array_equal(s_k, want.trace[:, 2]) and np.array_equal(m_t, want.trace[:, 6])
    if fp32:
        f32 = cheb.run_cpaa(dg, cheb.SolverConfig(c=C, eps=EPS, precision=32))
        rel = float(np.sum(np.abs(f32.ranks - want.ranks)) / np.sum(np.abs(want.ranks)))
        assert rel <= 1e-6, rel
    return want


def _threads():
    import bench
    return bench.host_threads()


def _check_power_and_apply(cheb, rg, dg, threads):
    want = rg.run_power(c=C, rounds=50, parallelism=threads)
    fast = cheb.run_power(dg, cheb.PowerConfig(c=C, rounds=50))
    assert float(np.max(np.abs(fast.ranks - want.ranks))) <= 1e-12
    exact = cheb.run_power(dg, cheb.PowerConfig(c=C, rounds=50, mode=cheb.MODE_BITEXACT))
    assert np.array_equal(exact.ranks, want.ranks)
    assert np.array_equal(np.array([r.l1_change for r in exact.trace]), want.trace[:, 4])
    rng = np.random.default_rng(7)
    x = rng.random(rg.n)
    y_ref = rg.transition_apply(x)
    assert np.array_equal(cheb.transition_apply(dg, x, mode=cheb.MODE_BITEXACT), y_ref)
    assert float(np.max(np.abs(cheb.transition_apply(dg, x) - y_ref))) <= 1e-12 * float(np.max(np.abs(y_ref)))


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_config_full_size_vs_reference(cheb, reference, name):
    rg = _reference_side(reference, name)
    dg, info = _device_side(name)
    _check_csr(rg, dg, info)
    _check_solves(cheb, rg, dg, _threads())
    _check_power_and_apply(cheb, rg, dg, _threads())
    nw, entries = _windows(dg)
    if name == "c3":  # the solves above ran the window schedule (24 windows), config 2 the plain one
        assert nw == 24 and entries > 0.5 * info["nnz"]
    else:
        assert nw == 0
    dg.free()


def test_config4_full_size_vs_reference(cheb, reference):
    """1.05 G CSR entries, int64 row pointers, x larger than L2: CSR bit-exact, FAST within
    1e-12 with the reference's top-100, BITEXACT bitwise (ranks and trace), fp32 within 1e-6."""
    rg = _reference_side(reference, "c4")
    dg, info = _device_side("c4")
    assert info["row_ptr_64"] == 1 and info["nnz"] > 1_000_000_000
    _check_csr(rg, dg, info)
    rg._csr = None
    gc.collect()
    want = _check_solves(cheb, rg, dg, _threads(), fp32=True)
    nw, entries = _windows(dg)  # ... through the window schedule: 64 windows, two thirds of the entries
    assert nw == 64 and entries > 0.6 * info["nnz"]
    # the mass ledger of the reference's own trace holds for ours too
    t = cheb.coefficients(C, 39)
    n = float(info["n"])
    partial = t.c0 / 2.0
    for k in range(39):
        partial += t.coeffs[k + 1]
        assert abs(want.trace[k, 2] - n * partial) <= n * 1e-12
    dg.free()


def test_config5_sampled_columns_vs_restated_loop(cheb, reference, oracle):
    """Batched R = 64 (K5): 4 of the 64 one-hot columns against the restated CPAA loop
    (T0 = e_seed) on the reference-built CSR; fp32 within 1e-6 relative L1."""
    import threading
    import bench
    rg = _reference_side(reference, "c5")
    dg, info = _device_side("c5")
    _check_csr(rg, dg, info)
    csr = rg.csr()
    seeds = bench.c5_seeds_from_degrees(csr.degrees, 64)
    res = cheb.run_cpaa_batch(dg, cheb.SolverConfig(c=C, eps=EPS), seeds=seeds)
    f32 = cheb.run_cpaa_batch(dg, cheb.SolverConfig(c=C, eps=EPS, precision=32), seeds=seeds)
    assert res.ranks.shape == (info["n"], 64)
    assert np.max(np.abs(res.ranks.sum(axis=0) - 1.0)) <= 1e-10
    cols = [0, 21, 42, 63]
    want = {}

    def one(r):
        p = np.zeros(csr.n)
        p[seeds[r]] = 1.0
        want[r] = oracle.run_cpaa(csr, 39, c=C, p=p).ranks
    th = [threading.Thread(target=one, args=(r,)) for r in cols]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in cols:
        err = float(np.max(np.abs(res.ranks[:, r] - want[r])))
        assert err <= 1e-12, (r, err)
        assert np.array_equal(top100(res.ranks[:, r]), top100(want[r])), r
        rel = float(np.sum(np.abs(f32.ranks[:, r] - want[r])) / np.sum(np.abs(want[r])))
        assert rel <= 1e-6, (r, rel)
    dg.free()

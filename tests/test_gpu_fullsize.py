"""Full-size parity (BASELINE.json configs 2 and 3) through size-independent properties:
CSR invariants of the device builder on the full graph, FAST vs BITEXACT agreement
(BITEXACT = the reference's arithmetic, bitwise-pinned on the fixtures), the mass ledger
S_k = n (c0/2 + sum c_i), unit total mass, top-100 stability, fp32 relative L1, batched
uniform column vs the scalar solve.  Inputs come from the same seeded generators as
bench.py."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
C = 0.85


def _build(cfg_name):
    import bench
    dg, info = bench.build_device(bench.CONFIGS[cfg_name], 0)
    return dg, info


def _csr_properties(g):
    off, nb, deg = g.offsets, g.neighbors, g.degrees
    n = g.n
    assert off[0] == 0 and off[-1] == nb.size and np.all(np.diff(off) == deg) and deg.min() >= 1
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    assert nb.min() >= 0 and nb.max() < n
    same = rows[1:] == rows[:-1]
    assert np.all(nb[1:][same] > nb[:-1][same])                      # sorted, no duplicates
    a = np.sort(rows * n + nb)
    b = np.sort(nb * n + rows)
    assert np.array_equal(a, b)                                       # symmetric
    assert nb.size == 2 * g.m - int(np.count_nonzero(nb == rows))     # entries = 2m - loops


def test_config2_full_size(cheb):
    dg, info = _build("c2")
    g = dg.download()
    _csr_properties(g)
    assert info["n"] == 1 << 20
    fast = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    exact = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, mode=cheb.MODE_BITEXACT))
    assert fast.rounds == 39 and exact.rounds == 39
    assert np.max(np.abs(fast.ranks - exact.ranks)) <= 1e-12
    top = lambda r: np.argsort(-r, kind="stable")[:100]  # noqa: E731
    assert np.array_equal(top(fast.ranks), top(exact.ranks))
    t = cheb.coefficients(C, 39)
    n = float(g.n)
    partial = t.c0 / 2.0
    for row in fast.trace:
        partial += t.coeffs[row.k]
        assert abs(row.S_k - n * partial) <= n * 1e-12                 # mass ledger
        assert abs(row.mass_T - n) <= n * 1e-12                        # T_k conserves mass
    assert abs(cheb.kahan_sum(fast.ranks) - 1.0) <= 1e-12
    f32 = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, precision=32))
    assert np.sum(np.abs(f32.ranks - exact.ranks)) / np.sum(exact.ranks) <= 1e-6
    # the 210-round Power reference and CPAA agree to the a-priori bound
    p = cheb.run_power(dg, cheb.PowerConfig(rounds=210))
    assert np.sum(np.abs(p.ranks - fast.ranks)) <= 1e-9
    dg.free()


def test_config3_full_size(cheb):
    dg, info = _build("c3")
    assert info["isolated_dropped"] > 0 and info["nnz"] > 100_000_000
    fast = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    again = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    assert np.array_equal(fast.ranks, again.ranks)                     # deterministic
    t = cheb.coefficients(C, 39)
    n = float(info["n"])
    partial = t.c0 / 2.0
    for row in fast.trace:
        partial += t.coeffs[row.k]
        assert abs(row.S_k - n * partial) <= n * 1e-12
    assert abs(cheb.kahan_sum(fast.ranks) - 1.0) <= 1e-12
    exact = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, mode=cheb.MODE_BITEXACT))
    assert np.max(np.abs(fast.ranks - exact.ranks)) <= 1e-12
    dg.free()


def test_config4_full_size(cheb):
    """1.05 B CSR entries, int64 row pointers, x larger than L2 (the L2 window path)."""
    dg, info = _build("c4")
    assert info["row_ptr_64"] == 1 and info["nnz"] > 1_000_000_000
    fast = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    again = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    assert fast.rounds == 39 and np.array_equal(fast.ranks, again.ranks)   # deterministic
    t = cheb.coefficients(C, 39)
    n = float(info["n"])
    partial = t.c0 / 2.0
    for row in fast.trace:
        partial += t.coeffs[row.k]
        assert abs(row.S_k - n * partial) <= n * 1e-12                      # mass ledger
    assert abs(cheb.kahan_sum(fast.ranks) - 1.0) <= 1e-12
    p = cheb.run_power(dg, cheb.PowerConfig(rounds=210))                  # independent solver
    assert np.sum(np.abs(p.ranks - fast.ranks)) <= 1e-9
    dg.free()


def test_config5_full_size(cheb):
    """Batched R = 64 (K5): every column is a distribution, and columns equal the scalar
    personalised solves (one-hot T_0) of their seeds."""
    import bench
    dg, info = _build("c5")
    seeds = bench.c5_seeds(dg, 64)
    res = cheb.run_cpaa_batch(dg, cheb.SolverConfig(eps=1e-10), seeds=seeds)
    assert res.ranks.shape == (info["n"], 64)
    sums = res.ranks.sum(axis=0)
    assert np.max(np.abs(sums - 1.0)) <= 1e-10
    for r in (0, 37):
        p = np.zeros(info["n"])
        p[seeds[r]] = 1.0
        single = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10, personalization=p))
        assert np.max(np.abs(single.ranks - res.ranks[:, r])) <= 1e-12
    # fp32 variant (fp32 storage, fp64 row sums): relative L1 <= 1e-6 per column
    f32 = cheb.run_cpaa_batch(dg, cheb.SolverConfig(eps=1e-10, precision=32), seeds=seeds)
    rel = np.sum(np.abs(f32.ranks - res.ranks), axis=0) / np.sum(np.abs(res.ranks), axis=0)
    assert rel.max() <= 1e-6, rel.max()
    dg.free()

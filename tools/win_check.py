"""Column windows of the hub rows (cheb_set_tuning "windows"): ranks with NW windows against
the plain schedule on the same graph (max |d|, top-100, determinism), per-term time of both.
Usage: python tools/win_check.py config [NW ...]   (config: small | c2 | c3 | c4 | c5)"""
import ctypes as C
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402
from paper_2112_01743_b200 import generate as Gen  # noqa: E402

cfg = sys.argv[1]
nws = [int(a) for a in sys.argv[2:]] or [32]
prec = int(os.environ.get("PREC", "64"))
lib = L.load()


def build():
    if cfg == "small":
        e = Gen.chung_lu_edges(1 << 17, 2.1, 2.0, 20000.0, 1_500_000, 5)
        return cheb.build_device_graph(e)
    return bench.build_device(bench.CONFIGS[cfg], 0)


def term_us(dg):
    opts = L.cheb_cpaa_opts()
    lib.cheb_cpaa_opts_default(C.byref(opts))
    opts.eps = 1e-10
    opts.precision = prec
    ms = (C.c_double * 64)()
    terms = C.c_int()
    res = []
    for _ in range(3):
        cheb.api._check(lib.cheb_cpaa_profile(dg.handle, C.byref(opts), ms, 64, C.byref(terms)))
        res.append(statistics.median([ms[i] for i in range(1, terms.value)]))
    return min(res) * 1e3


def top100(r):
    return np.lexsort((np.arange(r.size), -r))[:100]


base = None
for nw in [0] + nws:
    assert lib.cheb_set_tuning(b"windows", nw) == 0
    dg, info = build()
    sc = cheb.SolverConfig(eps=1e-10) if prec == 64 else cheb.SolverConfig(eps=1e-10, precision=32)
    a = cheb.run_cpaa(dg, sc)
    b = cheb.run_cpaa(dg, sc)
    det = bool(np.array_equal(a.ranks, b.ranks))
    t = term_us(dg)
    if base is None:
        base = a.ranks
        print(f"{cfg} fp{prec} windows=0   {t:9.1f} us/term  deterministic={det} n={info['n']} nnz={info['nnz']}", flush=True)
    else:
        d = float(np.max(np.abs(a.ranks - base)))
        same = bool(np.array_equal(top100(a.ranks), top100(base)))
        print(f"{cfg} fp{prec} windows={nw:<3d} {t:9.1f} us/term  deterministic={det} max|d|={d:.3e} "
              f"rel-L1={float(np.sum(np.abs(a.ranks - base)) / np.sum(np.abs(base))):.3e} top100 same={same}", flush=True)
    dg.free()
lib.cheb_set_tuning(b"windows", 0)

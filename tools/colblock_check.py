"""Column-blocked chunk schedule: FAST ranks with K = 1 (off) against K = 2, 3 on one config
(each K on its own device graph; the schedule is fixed when the view is built).
Reports max-abs difference, top-100 identity and the per-term time of each K.
Usage: python tools/colblock_check.py config [K ...]"""
import ctypes as C
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1]
Ks = [int(k) for k in sys.argv[2:]] or [1, 2, 3]
lib = L.load()
base = None
for K in Ks:
    cheb.api._check(lib.cheb_set_tuning(b"colblocks", K))
    dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
    r = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10))
    opts = L.cheb_cpaa_opts()
    lib.cheb_cpaa_opts_default(C.byref(opts))
    opts.eps = 1e-10
    ms = (C.c_double * 64)()
    terms = C.c_int()
    best = 1e30
    for _ in range(3):
        cheb.api._check(lib.cheb_cpaa_profile(dg.handle, C.byref(opts), ms, 64, C.byref(terms)))
        best = min(best, statistics.median([ms[i] for i in range(1, terms.value)]))
    top = np.lexsort((np.arange(r.ranks.size), -r.ranks))[:100]
    if base is None:
        base = (r.ranks.copy(), top)
        d = 0.0
        same = True
    else:
        d = float(np.max(np.abs(r.ranks - base[0])))
        same = bool(np.array_equal(top, base[1]))
    print(f"{cfg} K={K} term {best*1e3:8.1f} us  max|d|={d:.3e} top100_same={same} sum={r.ranks.sum():.15f}",
          flush=True)
    dg.free()

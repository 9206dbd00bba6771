"""Single vs double column-buffer term kernel on a config: FAST ranks of repeated solves
(determinism) and of both variants (must be bitwise equal).  Usage: python tools/nb_check.py cfg"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1]
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
res = {}
for nb in (2, 1, 1, 1):
    lib.cheb_set_tuning(b"colbufs", nb)
    r = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks
    res.setdefault(nb, []).append(r)
base = res[2][0]
for i, r in enumerate(res[1]):
    d = np.abs(r - base)
    print(f"{cfg} nb=1 run {i}: max|d| vs nb=2 {d.max():.3e}, differing entries {(d > 0).sum()}", flush=True)

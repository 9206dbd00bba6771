"""Batched (K5) solve time per column-block size: one call of cheb_cpaa_batch with the
config's 64 one-hot seeds, the device time of the whole call (all column blocks) from
cheb_last_timing.  Usage: python tools/batch_time.py [config] [precision]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 64
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
seeds = bench.c5_seeds_from_degrees(np.diff(dg.download().offsets), 64)
o = L.cheb_cpaa_opts()
lib.cheb_cpaa_opts_default(C.byref(o))
o.eps, o.precision, o.R = 1e-10, prec, 64
sp = seeds.ctypes.data_as(L.I64P)
ref = None
variants = [(64, 0), (64, 1), (96, 1), (48, 1), (96, 0)] if "sweep" in sys.argv else [(64, 0)]
for hub_mb, xpol in variants:
    blk = 64
    lib.cheb_set_tuning(b"spmm_hub_mb", hub_mb)
    lib.cheb_set_tuning(b"spmm_xpol", xpol)
    ts = []
    for i in range(3):
        cheb.api._check(lib.cheb_cpaa_batch(dg.handle, C.byref(o), sp, None, None, None, None))
        lm = C.c_double()
        lib.cheb_last_timing(dg.handle, C.byref(lm), None, None, None)
        ts.append(lm.value)
    res = cheb.run_cpaa_batch(dg, cheb.SolverConfig(eps=1e-10, precision=prec), seeds=seeds)
    if ref is None:
        ref = res.ranks
    err = float(np.max(np.abs(res.ranks - ref)))
    t = min(ts)
    print(f"{cfg} fp{prec} hub {hub_mb} MB xpol {xpol}: {t:8.1f} ms/solve {t/39:7.3f} ms/term "
          f"{info['nnz']*64*39/(t*1e-3)/1e9:8.1f} GTEPS(nnz*R)  max|diff vs block 64| {err:.2e}", flush=True)

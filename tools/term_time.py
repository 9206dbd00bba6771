"""Per-term time (median over the terms of 2 plain-launch solves, CUDA events around each
term) of the FAST term kernel on a config with the current environment's tuning.
Usage: python tools/term_time.py config [label]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else ""
prec = int(os.environ.get("PREC", "64"))
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
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
B = bench.algorithmic_bytes(info["n"], info["nnz"], 8 if info["row_ptr_64"] else 4, prec // 8)
t = min(res)
print(f"{cfg} fp{prec} {label:24s} {t*1e3:9.1f} us/term  {B/(t*1e-3)/1e9:7.1f} GB/s", flush=True)

"""Phase breakdown of the e2e path (reference-facing call with host buffers): upload of the
pinned int64 CSR, first solve (solver-view build + plain launches), repeated solve, ranks
read-back.  Usage: python tools/e2e_breakdown.py [config]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
pageable = "pageable" in sys.argv[2:]  # caller buffers as a C++ user holds them
fp32 = "fp32" in sys.argv[2:]
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
host = dg.download()
pin = (lambda a: a.copy()) if pageable else (lambda a: torch.from_numpy(a).pin_memory().numpy())
off = pin(host.offsets)
nb = pin(host.neighbors)
inv = pin(host.inv_degree)
ranks = torch.empty(host.n, dtype=torch.float64).pin_memory().numpy()
o = L.cheb_cpaa_opts()
lib.cheb_cpaa_opts_default(C.byref(o))
o.eps = 1e-10
if fp32:
    o.precision = 32
tr = (L.cheb_trace_row * 64)()
rounds, tot = C.c_int(), C.c_double()
for it in range(int(os.environ.get("ITERS", "4"))):
    t0 = time.perf_counter()
    h = C.c_void_p()
    cheb.api._check(lib.cheb_graph_upload_csr(off.ctypes.data_as(L.I64P), off.size, nb.ctypes.data_as(L.I64P),
                                              nb.size, host.degrees.ctypes.data_as(L.I64P), host.degrees.size,
                                              inv.ctypes.data_as(L.F64P), inv.size,
                                              host.n, host.m, 0, 0, int(info["row_ptr_64"]), C.byref(h)))
    t1 = time.perf_counter()
    cheb.api._check(lib.cheb_cpaa(h, C.byref(o), None, 0, ranks.ctypes.data_as(L.F64P), tr, C.byref(rounds),
                                  C.byref(tot)))
    t2 = time.perf_counter()
    lm = C.c_double()
    lib.cheb_last_timing(h, C.byref(lm), None, None, None)
    cheb.api._check(lib.cheb_cpaa(h, C.byref(o), None, 0, ranks.ctypes.data_as(L.F64P), tr, C.byref(rounds),
                                  C.byref(tot)))
    t3 = time.perf_counter()
    lib.cheb_graph_free(h)
    t4 = time.perf_counter()
    print(f"iter {it}: upload {1e3*(t1-t0):7.2f} ms | first solve {1e3*(t2-t1):7.2f} ms "
          f"(device loop {lm.value:6.2f}) | second solve {1e3*(t3-t2):7.2f} ms | free {1e3*(t4-t3):6.2f} ms")

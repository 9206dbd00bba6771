"""Graph-replayed solve time (device loop, cheb_last_timing) of a config under the current
environment's tuning.  Usage: python tools/solve_time.py config [label]"""
import ctypes as C
import os
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
sc = cheb.SolverConfig(eps=1e-10, precision=prec)
res = []
for i in range(6):
    cheb.run_cpaa(dg, sc)
    ms, per = C.c_double(), C.c_double()
    terms, launches = C.c_int(), C.c_int()
    cheb.api._check(lib.cheb_last_timing(dg.handle, C.byref(ms), C.byref(per), C.byref(terms), C.byref(launches)))
    if i >= 2:
        res.append(ms.value)
print(f"{cfg} fp{prec} {label:20s} solve {min(res):9.3f} ms  {min(res)/terms.value*1e3:9.1f} us/term  launches {launches.value}", flush=True)

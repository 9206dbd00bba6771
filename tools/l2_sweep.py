"""L2 policy sweep of the term kernel on one config (per-term time, CUDA events around each
term of a plain-launch solve): persisting-window size / hit ratio over the head of x, and
streaming (.cs) loads/stores of the per-row operands.  Usage: python tools/l2_sweep.py [config]
The nogather / skip / skipwarm / prefetch / streamcs knobs act only in the experiment build
(`touch paper_2112_01743_b200/csrc/term.cuh && make EXP=1`); the product build compiles them out."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
opts = L.cheb_cpaa_opts()
lib.cheb_cpaa_opts_default(C.byref(opts))
opts.eps = 1e-10
DEFAULTS = {"hot": -1, "l2win": 1, "pdl": 1, "l2win_mb": -1, "l2win_pct": 100, "streamcs": 0, "xout_hint": -1, "xdiscard": 1, "prefetch": 0, "nogather": 0, "skipwarm": 0}
print(f"{cfg} n={info['n']} nnz={info['nnz']}", flush=True)


def run(label, **kv):
    for k, v in kv.items():
        lib.cheb_set_tuning(k.encode(), v)
    ms = (C.c_double * 64)()
    terms = C.c_int()
    res = []
    for _ in range(2):
        cheb.api._check(lib.cheb_cpaa_profile(dg.handle, C.byref(opts), ms, 64, C.byref(terms)))
        res.append(statistics.median([ms[i] for i in range(1, terms.value)]))
    print(f"{label:34s} {min(res)*1e3:9.1f} us/term", flush=True)
    for k in kv:
        lib.cheb_set_tuning(k.encode(), DEFAULTS.get(k, 0))


run("default")
for P in (-1, -2, -3, -4):
    run(f"LSU L2 prefetch {-P} ahead", prefetch=P)
run("nogather", nogather=1)
run("nogather LSU prefetch 2", nogather=1, prefetch=-2)

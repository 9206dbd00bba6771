"""Kernel study: per-term time of the fused CPAA term kernel on a config under tuning
variants (hot-prefix size, gathers on/off).  Timing via cheb_cpaa_profile (CUDA events
around every term launch).  Usage: python tools/term_variants.py [config]
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

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 64
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
opts = L.cheb_cpaa_opts()
lib.cheb_cpaa_opts_default(C.byref(opts))
opts.eps = 1e-10
opts.precision = prec
B = bench.algorithmic_bytes(info["n"], info["nnz"], 8 if info["row_ptr_64"] else 4, prec // 8)
print(f"{cfg} n={info['n']} nnz={info['nnz']} maxdeg={info['max_degree']} bytes/term={B/1e6:.1f}MB fp{prec}")


def run(label, **kv):
    for k, v in kv.items():
        lib.cheb_set_tuning(k.encode(), v)
    ms = (C.c_double * 64)()
    terms = C.c_int()
    res = []
    for _ in range(3):
        cheb.api._check(lib.cheb_cpaa_profile(dg.handle, C.byref(opts), ms, 64, C.byref(terms)))
        res.append(statistics.median([ms[i] for i in range(1, terms.value)]))
    t = min(res)
    print(f"{label:28s} {t*1e3:8.1f} us/term  {B/(t*1e-3)/1e9:7.1f} GB/s  {info['nnz']/(t*1e-3)/1e9:7.1f} GTEPS")
    for k in kv:
        lib.cheb_set_tuning(k.encode(), {"hot": -1, "l2win": 1, "pdl": 1}.get(k, 0))


run("default")
run("hot=0 (all L2 gathers)", hot=0)
run("hot=4096", hot=4096)
run("no L2 window", l2win=0)
run("no gathers", nogather=1)
run("chunk tiles only", skip=2)
run("pack tiles only", skip=1)
run("chunk only, no gathers", skip=2, nogather=1)
run("pack only, no gathers", skip=1, nogather=1)
run("no PDL", pdl=0)

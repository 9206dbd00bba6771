"""validate (graph.cpp:123-186) at scale: the reference's (oracle/_ref, one host thread) vs
the device version (cheb_validate_csr, host arrays in, stats out) on a bench config's CSR.
Usage: python tools/validate_bench.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
g = dg.download()
for _ in range(2):
    t = time.perf_counter()
    st = cheb.validate(g)
    dt = time.perf_counter() - t
print(f"{cfg}: n={g.n} nnz={g.neighbors.size} device validate {dt * 1e3:.1f} ms (self_loops {st.self_loops})")
from oracle import CSR, Reference  # noqa: E402  (the reference, checker / baseline)
rg = Reference().graph_from_csr(CSR(g.n, g.m, g.offsets, g.neighbors, g.degrees, g.inv_degree, 0, 0, g.multi))
t = time.perf_counter()
rs = rg.validate()
print(f"{cfg}: reference validate {(time.perf_counter() - t) * 1e3:.1f} ms (self_loops {rs['self_loops']})")

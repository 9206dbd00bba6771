"""run_power (tol 1e-10 stop, max 1000 rounds) in BITEXACT and FAST vs the reference's
run_power (oracle/_ref, 1 thread) on gnp graphs.  Usage: python tools/power_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import generate as G  # noqa: E402

for n, p in ((20_000, 0.001), (100_000, 0.0001)):
    e = G.gnp_edges(n, p, 3)
    dg, info = cheb.build_device_graph(e)
    row = [f"n={info['n']:7d} nnz={info['nnz']:8d}"]
    for mode, name in ((cheb.MODE_BITEXACT, "bitexact"), (cheb.MODE_FAST, "fast")):
        cfg = cheb.PowerConfig(tol=1e-10, max_rounds=1000, mode=mode)
        r = cheb.run_power(dg, cfg)
        t = time.perf_counter()
        r = cheb.run_power(dg, cfg)
        row.append(f"{name} {(time.perf_counter() - t) * 1e3:8.2f} ms ({r.rounds} rounds)")
    from oracle import Reference
    rg = Reference().build_graph(e)
    t = time.perf_counter()
    rr = rg.run_power(tol=1e-10, max_rounds=1000, parallelism=1)
    row.append(f"reference(1 thread) {(time.perf_counter() - t) * 1e3:8.2f} ms ({rr.rounds} rounds)")
    print(" | ".join(row))

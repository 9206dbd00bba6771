"""Solve time of the BITEXACT and FAST schedules vs the reference (oracle/_ref, 1 thread) on
gnp graphs around the drop-in's Auto threshold (2^20 CSR entries).
Usage: python tools/mode_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import generate as G  # noqa: E402

for n, p in ((20_000, 0.001), (100_000, 0.0001), (400_000, 0.000025)):
    e = G.gnp_edges(n, p, 3)
    dg, info = cheb.build_device_graph(e)
    row = [f"n={info['n']:7d} nnz={info['nnz']:8d}"]
    for mode, name in ((cheb.MODE_BITEXACT, "bitexact"), (cheb.MODE_FAST, "fast")):
        cfg = cheb.SolverConfig(eps=1e-10, mode=mode)
        cheb.run_cpaa(dg, cfg)
        t = time.perf_counter()
        for _ in range(3):
            cheb.run_cpaa(dg, cfg)
        row.append(f"{name} {(time.perf_counter() - t) / 3 * 1e3:8.2f} ms")
    from oracle import Reference  # the reference (checker / baseline only)
    ref = Reference()
    rg = ref.build_graph(e)
    t = time.perf_counter()
    rg.run_cpaa(eps=1e-10, parallelism=1)
    row.append(f"reference(1 thread) {(time.perf_counter() - t) * 1e3:8.2f} ms")
    print(" | ".join(row))

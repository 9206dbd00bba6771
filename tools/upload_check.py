"""The uploaded handle (grouped permute + sort overlapping the neighbour copy) and the
device-built handle (K1) of the same graph have the same solver view: bitwise-equal FAST
ranks.  Usage: python tools/upload_check.py config"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
a = cheb.run_cpaa(dg, cheb.SolverConfig(eps=1e-10)).ranks
host = dg.download()
dg.free()
pin = lambda x: torch.from_numpy(x).pin_memory().numpy()  # noqa: E731
host.offsets, host.neighbors, host.inv_degree = pin(host.offsets), pin(host.neighbors), pin(host.inv_degree)
for i in range(3):
    t = time.perf_counter()
    h = cheb.upload(host, device=0, row_ptr_64=bool(info["row_ptr_64"]))
    t1 = time.perf_counter()
    b = cheb.run_cpaa(h, cheb.SolverConfig(eps=1e-10)).ranks
    t2 = time.perf_counter()
    h.free()
    print(f"{cfg}: upload {1e3*(t1-t):.1f} ms, solve {1e3*(t2-t1):.1f} ms, bitwise equal to K1 view: {np.array_equal(a, b)}",
          flush=True)

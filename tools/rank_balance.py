"""Row-partition balance on one B200: for G = 2, 4, 8 the config's graph is split by the
reference's cut rule over the degree-sorted relabel; per rank: rows, CSR
entries, hub rows, halo-push stores per term (and replicate-to-all), and the rank's mean term
time with the ranks' term kernels serialised (each timed on the whole GPU).  Usage:
python tools/rank_balance.py [config]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402
from paper_2112_01743_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
lib = L.load()
dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
host = dg.download()
dg.free()
print(f"{cfg}: n={info['n']} nnz={info['nnz']}", flush=True)
single = cheb.upload(host, device=0, row_ptr_64=bool(info["row_ptr_64"]))
ms = (C.c_double * 64)()
terms = C.c_int()
o = L.cheb_cpaa_opts()
lib.cheb_cpaa_opts_default(C.byref(o))
o.eps = 1e-10
cheb.api._check(lib.cheb_cpaa_profile(single.handle, C.byref(o), ms, 64, C.byref(terms)))
t1 = float(np.median([ms[i] for i in range(1, terms.value)]))
print(f"G=1: term {t1*1e3:.1f} us", flush=True)
single.free()
for G in (2, 4, 8):
    hs = [cheb.upload(host, device=0, row_ptr_64=bool(info["row_ptr_64"])) for _ in range(G)]
    grp = cheb.PartitionGroup(hs)
    rt = grp.rank_term_ms(cheb.SolverConfig(eps=1e-10))
    rows = []
    for r, h in enumerate(hs):
        lo, hi, nnz, mr = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        lib.cheb_graph_partition_info(h.handle, C.byref(lo), C.byref(hi), C.byref(nnz), C.byref(mr))
        bins = (C.c_int64 * 7)()
        lib.cheb_graph_view_bins(h.handle, None, bins, None)
        a, b = C.c_int64(), C.c_int64()
        lib.cheb_graph_exchange_info(h.handle, C.byref(a), C.byref(b))
        rows.append((r, hi.value - lo.value, nnz.value, bins[6], a.value, b.value, rt[r]))
    mx = max(x[6] for x in rows)
    print(f"G={G}: max rank term {mx*1e3:.1f} us (ideal {t1/G*1e3:.1f}); compute-only strong scaling {t1/mx:.2f}x", flush=True)
    for r, nr, nz, hub, halo, allst, t in rows:
        print(f"  rank {r}: rows {nr:9d} nnz {nz:11d} hub rows {hub:7d} push stores halo {halo:10d} "
              f"(all {allst:10d}, {halo/max(allst,1):.2f}) term {t*1e3:8.1f} us", flush=True)
    grp.close()
    for h in hs:
        h.free()

"""Graph ingest: the reference's load_edge_list (oracle/_ref, graph_io.cpp:50-70 + build_graph
+ validate, one host thread) against the device loader (file -> pinned ring -> GPU line
parse -> K1) on the same edge-list file of a bench config (default c2).  The file is written
once (page cache warm for both arms).  Usage: python tools/ingest_bench.py [config]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2112_01743_b200 as cheb  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[cfg_name]
edges = np.asarray(bench.make_edges_host(cfg))
edges = edges.reshape(-1, 2).astype(np.int64)
path = os.path.join(tempfile.mkdtemp(), f"{cfg_name}.txt")
t = time.perf_counter()
with open(path, "w") as f:
    f.write(f"# {cfg_name}: {edges.shape[0]} edges\n")
    np.savetxt(f, edges, fmt="%d %d")
size = os.path.getsize(path)
print(f"{cfg_name}: {edges.shape[0]} lines, {size/1e6:.1f} MB written in {time.perf_counter()-t:.1f} s")
opts = cheb.LoadOptions(drop_isolated=cfg.get("drop", False))

# device: file -> resident graph handle (what a solver needs)
for it in range(4):
    t = time.perf_counter()
    dg, st = cheb.load_device_graph(path, "edges", opts)
    dt = time.perf_counter() - t
    dg.free()
    print(f"device load_device_graph: {dt*1e3:8.1f} ms  ({size/dt/1e9:5.2f} GB/s of text, "
          f"{edges.shape[0]/dt/1e6:6.1f} M lines/s)  n={st.n} m={st.m}")
t = time.perf_counter()
lg = cheb.load_edge_list(path, opts)
print(f"device load_edge_list (+ host CSR download): {(time.perf_counter()-t)*1e3:8.1f} ms")

from oracle import Reference  # noqa: E402  (the reference arm; checker only)
ref = Reference()
t = time.perf_counter()
g, rst = ref.load(path, "edges", drop_isolated=opts.drop_isolated)
rt = time.perf_counter() - t
print(f"reference load_edge_list (1 host thread): {rt*1e3:8.1f} ms  ({size/rt/1e9:5.3f} GB/s)")
c = g.csr()
same = (np.array_equal(c.offsets, lg.graph.offsets) and np.array_equal(c.neighbors, lg.graph.neighbors)
        and rst["m"] == lg.stats.m and rst["self_loops"] == lg.stats.self_loops)
print(f"CSR + stats identical: {same}")
os.remove(path)

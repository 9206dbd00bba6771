"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref = the reference's
sources compiled unmodified).  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The .npz files are committed; the GPU box only reads them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import Reference  # noqa: E402

R = Reference()
C = 0.85


def path_edges(n):
    return np.array([[i, i + 1] for i in range(n - 1)], dtype=np.int64)


CASES = {
    # named fixtures of /root/reference/proj/tests/helpers.hpp:34-37
    "k2": (np.array([[0, 1]]), {}),
    "path3": (path_edges(3), {}),
    "star4": (np.array([[0, 1], [0, 2], [0, 3]]), {}),
    "cycle4": (R.ring_edges(4), {}),
    # build_graph edge cases (test_graph.cpp:35-91)
    "dup": (np.array([[0, 1], [1, 0], [1, 2]]), {}),
    "multi": (np.array([[0, 1], [1, 0], [0, 1], [1, 2]]), {"dedup": False}),
    "selfloop": (np.array([[0, 1], [0, 0], [1, 2], [2, 2]]), {}),
    "drop": (np.array([[0, 1], [3, 4], [4, 6], [6, 3]]), {"drop_isolated": True}),
    "nhint_drop": (np.array([[0, 1], [1, 2]]), {"drop_isolated": True, "n_hint": 6}),
    # random graphs used by the reference tests (test_cpaa.cpp:157-329)
    "gnp500": (R.gnp_edges(500, 0.012, 7), {}),
    "gnp2000": (R.gnp_edges(2000, 0.003, 3), {}),
    "star100": (R.star_edges(100), {}),
    "regular30": (R.regular_edges(30, 4), {}),
    # BASELINE config 1: gnp_edges(10000, 0.001, seed 1)
    "config1": (R.gnp_edges(10000, 0.001, 1), {}),
}

for name, (edges, opts) in CASES.items():
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    rg = R.build_graph(edges, **opts)
    g = rg.csr()
    out = dict(edges=edges, n=g.n, m=g.m, offsets=g.offsets, neighbors=g.neighbors,
               degrees=g.degrees, duplicates_removed=rg.duplicates_removed,
               isolated_dropped=rg.isolated_dropped, multi=int(g.multi))
    if g.n >= 1:
        for M in (12, 39):
            r = rg.run_cpaa(c=C, rounds=M)
            out[f"cpaa{M}_ranks"] = r.ranks
            out[f"cpaa{M}_S"] = r.trace[:, 2]
            out[f"cpaa{M}_massT"] = r.trace[:, 6]
            out[f"cpaa{M}_total"] = r.total_mass
        p = rg.run_power(c=C, rounds=210)
        out["power210_ranks"] = p.ranks
        out["power210_l1"] = p.trace[:, 4]
        x = np.linspace(-0.5, 1.5, g.n)
        out["tapply_x"] = x
        out["tapply_y"] = rg.transition_apply(x)
        if g.n <= 512:
            out["dense"] = rg.dense_direct_solve(C)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, g.n, g.m, g.neighbors.size)

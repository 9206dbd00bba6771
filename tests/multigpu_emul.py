"""TEST INFRASTRUCTURE: CPU emulation of the multi-GPU CPAA protocol with
torch.distributed gloo — the library's own partition plan (cheb_partition_plan, host C++),
the padded exchange layout, an all_gather of x_{k+1} per term, trace sums combined in
rank order, and the final padded gather + un-permute.  Numerics in numpy (fp64)."""
import numpy as np
import torch
import torch.distributed as dist


def emulate(rank, world, offsets, neighbors, c=0.85, M=39):
    from paper_2112_01743_b200 import coefficients
    from paper_2112_01743_b200.distributed import partition_plan
    n = offsets.size - 1
    deg = np.diff(offsets)
    order, cuts, mr = partition_plan(deg, world)
    new_of_old = np.empty(n, dtype=np.int64)
    new_of_old[order] = np.arange(n)
    slot = np.searchsorted(cuts, new_of_old, side="right") - 1
    pos = slot * mr + (new_of_old - cuts[slot])                     # padded position per old id
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    rows_old = order[lo:hi]
    # local CSR in new row order, columns renamed to padded positions (storage order kept)
    starts, ends = offsets[rows_old], offsets[rows_old + 1]
    ldeg = ends - starts
    cols = np.concatenate([pos[neighbors[s:e]] for s, e in zip(starts, ends)]) if hi > lo else np.zeros(0, np.int64)
    seg = np.concatenate([[0], np.cumsum(ldeg)])
    inv = 1.0 / ldeg
    t = coefficients(c, M)
    c0, ck = t.c0, t.coeffs

    def gather_slot(local):
        buf = np.zeros(mr)
        buf[: local.size] = local
        out = [torch.zeros(mr, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(buf))
        return torch.cat(out).numpy()

    def segsum(x):
        if cols.size == 0:
            return np.zeros(hi - lo)
        vals = x[cols]
        return np.add.reduceat(vals, seg[:-1]) if vals.size else np.zeros(hi - lo)

    T_prev = np.ones(hi - lo)
    T_curr = np.ones(hi - lo)
    acc = np.full(hi - lo, c0 / 2.0)
    x = gather_slot(T_curr * inv)
    trace = np.zeros((M, 2))
    for k in range(1, M + 1):
        s = segsum(x)
        tk = s if k == 1 else 2.0 * s - T_prev
        acc = acc + ck[k] * tk
        trace[k - 1] = (tk.sum(), acc.sum())
        T_prev, T_curr = T_curr, tk
        x = gather_slot(tk * inv)
    # trace: rank-ordered combine
    allt = [torch.zeros(M * 2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allt, torch.from_numpy(trace.ravel().copy()))
    glob = sum(a.numpy() for a in allt).reshape(M, 2)
    total = glob[-1, 1]
    full = gather_slot(acc / total)
    ranks = np.zeros(n)
    for r in range(world):
        cnt = int(cuts[r + 1] - cuts[r])
        ranks[order[cuts[r]:cuts[r] + cnt]] = full[r * mr: r * mr + cnt]
    return ranks, glob, (lo, hi, mr)

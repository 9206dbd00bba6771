"""TEST INFRASTRUCTURE: CPU emulation of the multi-GPU CPAA protocol with
torch.distributed gloo — the library's degree-sorted relabel (cheb_partition_plan's order),
the block-cyclic snake-order row partition (blocks of cheb_partition_block_rows() rows;
common.cuh part_owner / part_global), x in the global sorted order on every rank, an
all_gather of every rank's slot + un-shuffle per term (the NCCL exchange), trace sums
combined in rank order, and the final gather + un-permute.  Numerics in numpy (fp64)."""
import numpy as np
import torch
import torch.distributed as dist


def block_rows():
    from paper_2112_01743_b200 import _lib as L
    return int(L.load().cheb_partition_block_rows())


def part_owner(u, G, B):
    b = np.asarray(u) // B
    c = b // G
    j = b - c * G
    return np.where(c & 1, G - 1 - j, j)


def part_global(i, r, G, B):
    i = np.asarray(i)
    c = i // B
    j = np.where(c & 1, G - 1 - r, r)
    return (c * G + j) * B + i % B


def part_local(u, G, B):
    u = np.asarray(u)
    return (u // B // G) * B + u % B


def local_rows(n, r, G, B):
    """sorted rows owned by rank r, in local order"""
    u = np.arange(n)
    return u[part_owner(u, G, B) == r]


def emulate(rank, world, offsets, neighbors, c=0.85, M=39):
    from paper_2112_01743_b200 import coefficients
    from paper_2112_01743_b200.distributed import partition_plan
    n = offsets.size - 1
    deg = np.diff(offsets)
    B = block_rows()
    order, _, _ = partition_plan(deg, world)            # degree-descending relabel
    new_of_old = np.empty(n, dtype=np.int64)
    new_of_old[order] = np.arange(n)
    counts = [local_rows(n, r, world, B).size for r in range(world)]
    mr = max(counts)
    mine = local_rows(n, rank, world, B)
    assert np.array_equal(mine, part_global(np.arange(mine.size), rank, world, B))
    rows_old = order[mine]
    starts, ends = offsets[rows_old], offsets[rows_old + 1]
    ldeg = ends - starts
    nl = mine.size
    cols = np.concatenate([new_of_old[neighbors[s:e]] for s, e in zip(starts, ends)]) if nl else np.zeros(0, np.int64)
    seg = np.concatenate([[0], np.cumsum(ldeg)])
    inv = 1.0 / ldeg
    t = coefficients(c, M)
    c0, ck = t.c0, t.coeffs
    u_all = np.arange(n)
    src = part_owner(u_all, world, B) * mr + part_local(u_all, world, B)

    def exchange(local):
        buf = np.zeros(mr)
        buf[: local.size] = local
        out = [torch.zeros(mr, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(buf))
        return torch.cat(out).numpy()[src]             # global sorted order

    def segsum(x):
        if cols.size == 0:
            return np.zeros(nl)
        return np.add.reduceat(x[cols], seg[:-1])

    T_prev = np.ones(nl)
    T_curr = np.ones(nl)
    acc = np.full(nl, c0 / 2.0)
    x = exchange(T_curr * inv)
    trace = np.zeros((M, 2))
    for k in range(1, M + 1):
        s = segsum(x)
        tk = s if k == 1 else 2.0 * s - T_prev
        acc = acc + ck[k] * tk
        trace[k - 1] = (tk.sum(), acc.sum())
        T_prev, T_curr = T_curr, tk
        x = exchange(tk * inv)
    allt = [torch.zeros(M * 2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allt, torch.from_numpy(trace.ravel().copy()))
    glob = sum(a.numpy() for a in allt).reshape(M, 2)
    total = glob[-1, 1]
    full = exchange(acc / total)
    ranks = np.zeros(n)
    ranks[order] = full
    return ranks, glob, (nl, mr, counts)

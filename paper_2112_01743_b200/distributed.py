"""Multi-GPU plumbing: one process per GPU, an NCCL communicator created by the library
(cheb_comm_create) from a unique id that rank 0 draws and torch.distributed broadcasts, or
the fused push exchange (PeerExchange).  Attaching either to a graph handle makes cheb_cpaa a
collective over the ranks; the rows are split block-cyclically in snake order
over the degree-sorted relabel (cheb_partition_block_rows rows per block)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import _check, DeviceGraph


def partition_plan(degrees, G: int):
    """cheb_partition_plan: (order new->old = the degree-descending relabel, cuts[G+1] = the
    reference's partition_vertices rule on it, max_rows).  The device partition uses the
    relabel with block-cyclic ownership (common.cuh part_owner), not the cuts."""
    deg = np.ascontiguousarray(degrees, dtype=np.int64)
    n = deg.size
    order = np.zeros(n, dtype=np.int64)
    cuts = np.zeros(G + 1, dtype=np.int64)
    mr = C.c_int64()
    _check(L.load().cheb_partition_plan(deg.ctypes.data_as(L.I64P), n, G, order.ctypes.data_as(L.I64P),
                                        cuts.ctypes.data_as(L.I64P), C.byref(mr)))
    return order, cuts, int(mr.value)


class Communicator:
    """NCCL communicator over the ranks of a torch.distributed process group."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch
        import torch.distributed as dist
        lib = L.load()
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _check(lib.cheb_nccl_unique_id(uid, 128))
        if world > 1:
            backend = dist.get_backend(group)
            dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
            dist.broadcast(t, src=0, group=group)
            uid = (C.c_ubyte * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        _check(lib.cheb_comm_create(uid, world, rank, device, C.byref(h)))
        self.handle, self.rank, self.world, self.device = h, rank, world, device

    def attach(self, dg: DeviceGraph):
        _check(L.load().cheb_graph_attach_comm(dg.handle, self.handle))

    def close(self):
        if self.handle:
            L.load().cheb_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerExchange:
    """Fused push exchange over the ranks of a torch.distributed process group (one process
    per GPU): every rank exports its exchange buffers as CUDA IPC handles,
    the handles are all-gathered, and each rank maps its peers' buffers.  After ``attach``
    the term kernels store x_{k+1} straight into every peer's buffer (NVLink), with a flag
    barrier per term instead of an NCCL all-gather."""

    def __init__(self, dg: DeviceGraph, rank: int, world: int, group=None):
        lib = L.load()
        mine = (C.c_ubyte * L.PEER_EXPORT_BYTES)()
        rc = lib.cheb_peer_export(dg.handle, world, rank, mine, L.PEER_EXPORT_BYTES)
        err = None if rc == 0 else lib.cheb_last_error().decode()
        # every rank reaches every collective, even after a local failure, so a failing rank
        # cannot leave its peers blocked; all ranks then raise (or succeed) together
        allb = self._all_gather(None if err else bytes(mine), world, group)
        bad = [r for r, b in enumerate(allb) if b is None]
        if not bad:
            buf = (C.c_ubyte * (L.PEER_EXPORT_BYTES * world)).from_buffer_copy(b"".join(allb))
            rc = lib.cheb_peer_import(dg.handle, buf, L.PEER_EXPORT_BYTES)
            err = None if rc == 0 else lib.cheb_last_error().decode()
            bad = [r for r, ok in enumerate(self._all_gather(err is None, world, group)) if not ok]
        if bad:
            lib.cheb_peer_detach(dg.handle)
            raise RuntimeError(f"push exchange unavailable on ranks {bad}" + (f": {err}" if err else ""))
        self.dg, self.rank, self.world = dg, rank, world

    @staticmethod
    def _all_gather(obj, world, group):
        if world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * world
        dist.all_gather_object(out, obj, group=group)
        return out

    def detach(self):
        if self.dg is not None and self.dg.handle:
            _check(L.load().cheb_peer_detach(self.dg.handle))
        self.dg = None


def partition_info(dg: DeviceGraph) -> dict:
    """This rank's share of the block-cyclic row partition: rows, CSR entries, the largest
    rank's row count, and the halo-push stores per term (vs replicate-to-all)."""
    lo, hi, nnz, mr = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(L.load().cheb_graph_partition_info(dg.handle, C.byref(lo), C.byref(hi), C.byref(nnz), C.byref(mr)))
    a, b = C.c_int64(), C.c_int64()
    _check(L.load().cheb_graph_exchange_info(dg.handle, C.byref(a), C.byref(b)))
    return {"rows": hi.value - lo.value, "nnz_local": nnz.value, "max_rows": mr.value,
            "halo_stores": a.value, "all_stores": b.value}

"""Synthetic graph inputs (generate.hpp:27-40 of the reference, plus the configs' R-MAT /
Chung-Lu generators).  Host outputs are numpy (E, 2) arrays; device outputs are
``DeviceEdges`` owning a cudaMalloc'ed int32 pair buffer that the K1 builder consumes
without a host round trip."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import DomainError, _STATUS, Error


def _check(rc: int):
    if rc:
        raise _STATUS.get(rc, Error)(L.load().cheb_gen_last_error().decode())


def _host_i64(fn, *args) -> np.ndarray:
    lib = L.load()
    ptr, cnt = L.I64P(), C.c_int64()
    _check(fn(*args, C.byref(ptr), C.byref(cnt)))
    try:
        if cnt.value == 0:
            return np.zeros((0, 2), dtype=np.int64)
        return np.ctypeslib.as_array(ptr, shape=(cnt.value * 2,)).copy().reshape(-1, 2)
    finally:
        lib.cheb_free(ptr)


def ring_edges(n: int) -> np.ndarray:
    return _host_i64(L.load().cheb_gen_ring, n)


def star_edges(n: int) -> np.ndarray:
    return _host_i64(L.load().cheb_gen_star, n)


def regular_edges(n: int, k: int) -> np.ndarray:
    return _host_i64(L.load().cheb_gen_regular, n, k)


def gnp_edges(n: int, p: float, seed: int) -> np.ndarray:
    return _host_i64(L.load().cheb_gen_gnp, n, p, seed)


class DeviceEdges:
    """E int32 (u, v) pairs resident on a GPU (owned)."""

    def __init__(self, ptr: int, count: int, device: int):
        self.ptr, self.count, self.device = ptr, count, device

    def free(self):
        if self.ptr:
            L.load().cheb_device_free(C.c_void_p(self.ptr), self.device)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _gen32(fn, args, device):
    lib = L.load()
    ptr, cnt = C.c_void_p(), C.c_int64()
    on_dev = device is not None
    _check(fn(*args, int(on_dev), int(device or 0), C.byref(ptr), C.byref(cnt)))
    if on_dev:
        return DeviceEdges(ptr.value or 0, cnt.value, int(device))
    try:
        if cnt.value == 0:
            return np.zeros((0, 2), dtype=np.int32)
        buf = C.cast(ptr, C.POINTER(C.c_int32))
        return np.ctypeslib.as_array(buf, shape=(cnt.value * 2,)).copy().reshape(-1, 2)
    finally:
        lib.cheb_free(ptr)


def rmat_edges(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
               c: float = 0.19, seed: int = 1, device=None):
    """R-MAT, randomly relabelled, self-loops removed (configs 3/4)."""
    return _gen32(L.load().cheb_gen_rmat, (scale, edge_factor, a, b, c, seed), device)


def chung_lu_edges(n: int, gamma: float = 2.1, wmin: float = 2.0, wmax: float = 50000.0,
                   draws: int = 10_485_760, seed: int = 1, device=None):
    """Chung-Lu power-law graph, self-loops removed, isolated vertices rewired (configs 2/5)."""
    return _gen32(L.load().cheb_gen_chung_lu, (n, gamma, wmin, wmax, draws, seed), device)

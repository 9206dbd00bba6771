"""TEST INFRASTRUCTURE — ctypes bindings for the two CPU checkers.

* ``Oracle``    : our plain-C restatement (oracle/cpaa_oracle.c -> oracle/lib/liboracle.so)
* ``Reference`` : the reference's own sources compiled unmodified
                  (oracle/Makefile -> oracle/_ref/libchebpr_ref.so)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package.  The
product (``paper_2112_01743_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchebpr_ref.so")

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)

STATUS_NAMES = {1: "ValidationError", 2: "DomainError", 3: "NumericError",
                4: "InvalidArgument", 5: "CapacityError", 8: "ParseError", 9: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


def _p(a: np.ndarray | None, ty=F64P):
    if a is None:
        return None
    return a.ctypes.data_as(ty)


@dataclass
class CSR:
    n: int
    m: int
    offsets: np.ndarray
    neighbors: np.ndarray
    degrees: np.ndarray
    inv_degree: np.ndarray
    duplicates_removed: int = 0
    isolated_dropped: int = 0
    multi: bool = False


@dataclass
class Result:
    ranks: np.ndarray
    trace: np.ndarray           # rounds x 10: k,c_k,S_k,residual,l1,elapsed,mass_T,err,err_l1,0
    rounds: int
    total_mass: float
    wall_ms: float = 0.0


def edges_array(edges) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    return a


class Oracle:
    """Plain-C restatement (bit-identical to the reference; pinned in tests/test_oracle.py)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.or_last_error.restype = C.c_char_p
        L.or_kahan_sum.restype = C.c_double
        L.or_kahan_sum.argtypes = [F64P, C.c_int64]
        L.or_coefficients.argtypes = [C.c_double, C.c_int, F64P, F64P, F64P]
        L.or_plan_iterations.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int), F64P]
        L.or_err_bound.argtypes = [C.c_double, C.c_int, F64P]
        L.or_gnp_edges.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.POINTER(I64P), I64P]
        L.or_build_graph.argtypes = [I64P, C.c_int64, C.c_int, C.c_int, C.c_int64, I64P, I64P,
                                     C.POINTER(I64P), C.POINTER(I64P), C.POINTER(I64P),
                                     C.POINTER(F64P), I64P, I64P]
        L.or_transition_apply.argtypes = [C.c_int64, I64P, I64P, F64P, F64P, F64P]
        L.or_partition_vertices.argtypes = [C.c_int64, I64P, C.c_int, I64P]
        L.or_run_cpaa.argtypes = [C.c_int64, I64P, I64P, F64P, C.c_double, C.c_int, F64P, F64P,
                                  F64P, F64P]
        L.or_run_power.argtypes = [C.c_int64, I64P, I64P, F64P, C.c_double, C.c_int, C.c_double,
                                   C.c_int, F64P, F64P, C.POINTER(C.c_int), F64P]
        L.or_free.argtypes = [C.c_void_p]
        L.or_rmat_edges.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                    C.POINTER(I64P), I64P]
        L.or_chung_lu_edges.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64,
                                        C.c_uint64, C.POINTER(I64P), I64P]

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.or_last_error().decode())

    def kahan_sum(self, x: np.ndarray) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.lib.or_kahan_sum(_p(x), x.size)

    def coefficients(self, c: float, M: int):
        out = np.zeros(M + 1 if M >= 0 else 1)
        b, c0 = C.c_double(), C.c_double()
        self._check(self.lib.or_coefficients(c, M, _p(out), C.byref(b), C.byref(c0)))
        return out, b.value, c0.value

    def plan_iterations(self, c: float, eps: float):
        M, pe = C.c_int(), C.c_double()
        self._check(self.lib.or_plan_iterations(c, eps, C.byref(M), C.byref(pe)))
        return M.value, pe.value

    def err_bound(self, c: float, M: int) -> float:
        o = C.c_double()
        self._check(self.lib.or_err_bound(c, M, C.byref(o)))
        return o.value

    def gnp_edges(self, n: int, p: float, seed: int) -> np.ndarray:
        ptr, cnt = I64P(), C.c_int64()
        self._check(self.lib.or_gnp_edges(n, p, seed, C.byref(ptr), C.byref(cnt)))
        out = np.ctypeslib.as_array(ptr, shape=(max(cnt.value, 1) * 2,))[: cnt.value * 2].copy()
        self.lib.or_free(ptr)
        return out.reshape(-1, 2)

    def _take_edges(self, ptr, cnt) -> np.ndarray:
        try:
            if cnt.value == 0:
                return np.zeros((0, 2), dtype=np.int64)
            return np.ctypeslib.as_array(ptr, shape=(cnt.value * 2,)).copy().reshape(-1, 2)
        finally:
            self.lib.or_free(ptr)

    def rmat_edges(self, scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                   c: float = 0.19, seed: int = 1) -> np.ndarray:
        """Configs 3/4 edge list (oracle/synth_gen.c), int64 (E, 2)."""
        ptr, cnt = I64P(), C.c_int64()
        self._check(self.lib.or_rmat_edges(scale, edge_factor, a, b, c, seed, C.byref(ptr), C.byref(cnt)))
        return self._take_edges(ptr, cnt)

    def chung_lu_edges(self, n: int, gamma: float = 2.1, wmin: float = 2.0, wmax: float = 50000.0,
                       draws: int = 10_485_760, seed: int = 1) -> np.ndarray:
        """Configs 2/5 edge list (oracle/synth_gen.c), int64 (E, 2)."""
        ptr, cnt = I64P(), C.c_int64()
        self._check(self.lib.or_chung_lu_edges(n, gamma, wmin, wmax, draws, seed, C.byref(ptr), C.byref(cnt)))
        return self._take_edges(ptr, cnt)

    def build_graph(self, edges, dedup=True, drop_isolated=False, n_hint=0) -> CSR:
        e = edges_array(edges)
        n, m, d, dr = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        po, pn, pd, pi = I64P(), I64P(), I64P(), F64P()
        self._check(self.lib.or_build_graph(_p(e, I64P), e.shape[0], int(dedup), int(drop_isolated),
                                            n_hint, C.byref(n), C.byref(m), C.byref(po),
                                            C.byref(pn), C.byref(pd), C.byref(pi), C.byref(d),
                                            C.byref(dr)))
        nn = n.value

        def take(ptr, cnt, dt):
            if cnt == 0:
                out = np.zeros(0, dtype=dt)
            else:
                out = np.ctypeslib.as_array(ptr, shape=(cnt,)).copy()
            self.lib.or_free(ptr)
            return out

        off = take(po, nn + 1, np.int64)
        nb = take(pn, int(off[-1]) if nn >= 0 else 0, np.int64)
        deg = take(pd, nn, np.int64)
        inv = take(pi, nn, np.float64)
        return CSR(nn, m.value, off, nb, deg, inv, d.value, dr.value, not dedup)

    def transition_apply(self, g: CSR, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(g.n)
        self.lib.or_transition_apply(g.n, _p(g.offsets, I64P), _p(g.neighbors, I64P),
                                     _p(g.inv_degree), _p(x), _p(y))
        return y

    def partition_vertices(self, g: CSR, K: int) -> np.ndarray:
        cuts = np.zeros(K + 1, dtype=np.int64)
        self._check(self.lib.or_partition_vertices(g.n, _p(g.degrees, I64P), K, _p(cuts, I64P)))
        return cuts

    def run_cpaa(self, g: CSR, M: int, c: float = 0.85, p: np.ndarray | None = None) -> Result:
        ranks = np.zeros(g.n)
        trace = np.zeros((max(M, 1), 10))
        tm = C.c_double()
        pp = None if p is None else np.ascontiguousarray(p, dtype=np.float64)
        self._check(self.lib.or_run_cpaa(g.n, _p(g.offsets, I64P), _p(g.neighbors, I64P),
                                         _p(g.inv_degree), c, M, _p(pp), _p(ranks), _p(trace),
                                         C.byref(tm)))
        return Result(ranks, trace[:M], M, tm.value)

    def run_power(self, g: CSR, c: float = 0.85, rounds: int = -1, tol: float = -1.0,
                  max_rounds: int = 60) -> Result:
        ranks = np.zeros(g.n)
        budget = rounds if rounds >= 0 else max_rounds
        trace = np.zeros((max(budget, 1), 10))
        r, tm = C.c_int(), C.c_double()
        self._check(self.lib.or_run_power(g.n, _p(g.offsets, I64P), _p(g.neighbors, I64P),
                                          _p(g.inv_degree), c, rounds, tol, max_rounds, _p(ranks),
                                          _p(trace), C.byref(r), C.byref(tm)))
        return Result(ranks, trace[: r.value], r.value, tm.value)


class Reference:
    """The reference library itself (compiled unmodified by oracle/Makefile)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        for name in ("ref_gnp_edges",):
            getattr(L, name).argtypes = [C.c_int64, C.c_double, C.c_uint64, C.POINTER(I64P), I64P]
        L.ref_ring_edges.argtypes = [C.c_int64, C.POINTER(I64P), I64P]
        L.ref_star_edges.argtypes = [C.c_int64, C.POINTER(I64P), I64P]
        L.ref_regular_edges.argtypes = [C.c_int64, C.c_int64, C.POINTER(I64P), I64P]
        L.ref_build_graph.argtypes = [I64P, C.c_int64, C.c_int, C.c_int, C.c_int64,
                                      C.POINTER(C.c_void_p), I64P]
        L.ref_graph_from_arrays.restype = C.c_void_p
        L.ref_graph_from_arrays.argtypes = [C.c_int64, C.c_int64, I64P, C.c_int64, I64P, C.c_int64,
                                            I64P, C.c_int64, F64P, C.c_int64, C.c_int]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_get.argtypes = [C.c_void_p, I64P, I64P, I64P, F64P]
        L.ref_validate.argtypes = [C.c_void_p, I64P]
        run_args = [C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, F64P, F64P,
                    F64P, C.POINTER(C.c_int), F64P, F64P]
        L.ref_run_cpaa.argtypes = run_args
        L.ref_run_power.argtypes = run_args
        L.ref_transition_apply.argtypes = [C.c_void_p, F64P, C.c_int64, F64P]
        L.ref_staged_run.argtypes = [C.c_void_p, C.c_double, C.c_int, F64P, F64P]
        L.ref_dense_direct_solve.argtypes = [C.c_void_p, C.c_double, F64P]
        L.ref_coefficients.argtypes = [C.c_double, C.c_int, F64P, F64P, F64P]
        L.ref_plan_iterations.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int), F64P]
        L.ref_err_bound.argtypes = [C.c_double, C.c_int, F64P]
        L.ref_partition_vertices.argtypes = [C.c_void_p, C.c_int, I64P]
        L.ref_load.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p), I64P,
                               C.POINTER(C.c_double)]
        L.ref_solve_to_csv.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                       C.c_char_p, C.c_char_p]
        L.ref_write_edges.argtypes = [I64P, C.c_int64, C.c_char_p, C.c_char_p]
        L.ref_kahan_sum.restype = C.c_double
        L.ref_kahan_sum.argtypes = [F64P, C.c_int64]

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _edges(self, fn, *args) -> np.ndarray:
        ptr, cnt = I64P(), C.c_int64()
        self._check(fn(*args, C.byref(ptr), C.byref(cnt)))
        out = np.ctypeslib.as_array(ptr, shape=(max(cnt.value, 1) * 2,))[: cnt.value * 2].copy()
        self.lib.ref_free(ptr)
        return out.reshape(-1, 2)

    def gnp_edges(self, n, p, seed):
        return self._edges(self.lib.ref_gnp_edges, n, p, seed)

    def ring_edges(self, n):
        return self._edges(self.lib.ref_ring_edges, n)

    def star_edges(self, n):
        return self._edges(self.lib.ref_star_edges, n)

    def regular_edges(self, n, k):
        return self._edges(self.lib.ref_regular_edges, n, k)

    def build_graph(self, edges, dedup=True, drop_isolated=False, n_hint=0) -> "RefGraph":
        e = edges_array(edges)
        h = C.c_void_p()
        st = np.zeros(5, dtype=np.int64)
        self._check(self.lib.ref_build_graph(_p(e, I64P), e.shape[0], int(dedup), int(drop_isolated),
                                             n_hint, C.byref(h), _p(st, I64P)))
        return RefGraph(self, h, *[int(v) for v in st], multi=not dedup)

    def graph_from_csr(self, g: CSR) -> "RefGraph":
        h = self.lib.ref_graph_from_arrays(g.n, g.m, _p(g.offsets, I64P), g.offsets.size,
                                           _p(g.neighbors, I64P), g.neighbors.size,
                                           _p(g.degrees, I64P), g.degrees.size, _p(g.inv_degree),
                                           g.inv_degree.size, int(g.multi))
        return RefGraph(self, C.c_void_p(h), g.n, g.m, g.neighbors.size, 0, 0, multi=g.multi)

    def load(self, path, fmt="edges", dedup=True, drop_isolated=False, symmetrize=False):
        """The reference's own load_edge_list / load_matrix_market (graph_io.cpp:50-174).
        Returns (RefGraph, stats dict); raises OracleError(code, message) like the C++."""
        h = C.c_void_p()
        st = np.zeros(8, dtype=np.int64)
        avg = C.c_double()
        self._check(self.lib.ref_load(os.fsencode(path), 0 if fmt == "edges" else 1, int(dedup),
                                      int(drop_isolated), int(symmetrize), C.byref(h), _p(st, I64P),
                                      C.byref(avg)))
        stats = dict(n=int(st[0]), m=int(st[1]), min_degree=int(st[2]), max_degree=int(st[3]),
                     self_loops=int(st[4]), duplicates_removed=int(st[5]), isolated_dropped=int(st[6]),
                     avg_degree=avg.value)
        return RefGraph(self, h, int(st[0]), int(st[1]), int(st[7]), int(st[5]), int(st[6]), multi=not dedup), stats

    def coefficients(self, c, M):
        out = np.zeros(M + 1)
        b, c0 = C.c_double(), C.c_double()
        self._check(self.lib.ref_coefficients(c, M, _p(out), C.byref(b), C.byref(c0)))
        return out, b.value, c0.value

    def plan_iterations(self, c, eps):
        M, pe = C.c_int(), C.c_double()
        self._check(self.lib.ref_plan_iterations(c, eps, C.byref(M), C.byref(pe)))
        return M.value, pe.value

    def err_bound(self, c, M):
        o = C.c_double()
        self._check(self.lib.ref_err_bound(c, M, C.byref(o)))
        return o.value

    def kahan_sum(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.lib.ref_kahan_sum(_p(x), x.size)

    def write_edges(self, edges, path: str, comment: str):
        """The reference's write_edge_list (generate.cpp:89-97)."""
        e = edges_array(edges)
        self._check(self.lib.ref_write_edges(_p(e, I64P), e.shape[0], os.fsencode(path), comment.encode()))


@dataclass
class RefGraph:
    ref: Reference
    handle: C.c_void_p
    n: int
    m: int
    nnz: int
    duplicates_removed: int
    isolated_dropped: int
    multi: bool = False
    _csr: CSR | None = field(default=None, repr=False)

    def __del__(self):
        try:
            if self.handle:
                self.ref.lib.ref_graph_free(self.handle)
                self.handle = None
        except Exception:
            pass

    def csr(self) -> CSR:
        if self._csr is None:
            off = np.zeros(self.n + 1, dtype=np.int64)
            nb = np.zeros(max(self.nnz, 1), dtype=np.int64)
            deg = np.zeros(max(self.n, 1), dtype=np.int64)
            inv = np.zeros(max(self.n, 1))
            self.ref.lib.ref_graph_get(self.handle, _p(off, I64P), _p(nb, I64P), _p(deg, I64P), _p(inv))
            self._csr = CSR(self.n, self.m, off, nb[: self.nnz], deg[: self.n], inv[: self.n],
                            self.duplicates_removed, self.isolated_dropped, self.multi)
        return self._csr

    def validate(self):
        st = np.zeros(5, dtype=np.int64)
        self.ref._check(self.ref.lib.ref_validate(self.handle, _p(st, I64P)))
        return dict(n=int(st[0]), m=int(st[1]), min_degree=int(st[2]), max_degree=int(st[3]),
                    self_loops=int(st[4]))

    def _run(self, fn, c, rounds, eps_or_tol, max_rounds, parallelism, reference):
        budget = max(rounds if rounds >= 0 else max_rounds, 1)
        if fn is self.ref.lib.ref_run_cpaa and rounds < 0 and eps_or_tol > 0:
            budget = max(budget, 60)
        ranks = np.zeros(self.n)
        trace = np.zeros((budget + 1, 10))
        r, tm, wall = C.c_int(), C.c_double(), C.c_double()
        refp = None if reference is None else np.ascontiguousarray(reference, dtype=np.float64)
        self.ref._check(fn(self.handle, c, rounds, eps_or_tol, max_rounds, parallelism, _p(refp),
                           _p(ranks), _p(trace), C.byref(r), C.byref(tm), C.byref(wall)))
        return Result(ranks, trace[: r.value], r.value, tm.value, wall.value)

    def run_cpaa(self, c=0.85, rounds=-1, eps=-1.0, max_rounds=60, parallelism=1, reference=None):
        return self._run(self.ref.lib.ref_run_cpaa, c, rounds, eps, max_rounds, parallelism, reference)

    def run_power(self, c=0.85, rounds=-1, tol=-1.0, max_rounds=60, parallelism=1, reference=None):
        return self._run(self.ref.lib.ref_run_power, c, rounds, tol, max_rounds, parallelism, reference)

    def solve_to_csv(self, algo="cpaa", c=0.85, rounds=-1, eps=-1.0, max_rounds=60, ranks_path="",
                     trace_path=""):
        """run_cpaa / run_power, then the reference's own CSV writers (src/csv.cpp)."""
        self.ref._check(self.ref.lib.ref_solve_to_csv(self.handle, 0 if algo == "cpaa" else 1, c, rounds, eps,
                                                      max_rounds, os.fsencode(ranks_path), os.fsencode(trace_path)))

    def transition_apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        self.ref._check(self.ref.lib.ref_transition_apply(self.handle, _p(x), x.size, _p(y)))
        return y

    def staged_run(self, c, M):
        acc = np.zeros(self.n)
        tot = C.c_double()
        self.ref._check(self.ref.lib.ref_staged_run(self.handle, c, M, _p(acc), C.byref(tot)))
        return acc, tot.value

    def dense_direct_solve(self, c=0.85):
        out = np.zeros(self.n)
        self.ref._check(self.ref.lib.ref_dense_direct_solve(self.handle, c, _p(out)))
        return out

    def partition_vertices(self, K):
        cuts = np.zeros(K + 1, dtype=np.int64)
        self.ref._check(self.ref.lib.ref_partition_vertices(self.handle, K, _p(cuts, I64P)))
        return cuts

"""Python mirror of the reference's drop-in API (/root/reference/proj/include/chebpr/).

Same names, argument meaning and error behaviour as the reference's C++ headers
(graph.hpp, cpaa.hpp, power.hpp, coefficients.hpp, errors.hpp); every call goes
through the C-ABI of libchebpr_b200.so (include/chebpr_cuda.h) — the CUDA path is
the only path.  Additive options (``mode``, ``precision``, ``device``,
``personalization``) default to the reference's behaviour.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

# ---------------------------------------------------------------------------
# errors.hpp:11-33
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    """chebpr::Error"""


class ParseError(Error):
    pass


class ValidationError(Error):
    pass


class DomainError(Error):
    pass


class NumericError(Error):
    pass


class CapacityError(Error):
    pass


class CudaError(Error):
    """CUDA/NCCL failure inside the library (new)."""


InvalidArgument = ValueError  # std::invalid_argument

_STATUS = {1: ValidationError, 2: DomainError, 3: NumericError, 4: ValueError,
           5: CapacityError, 6: CudaError, 7: CudaError, 8: ParseError}

MODE_FAST, MODE_BITEXACT = 0, 1


def _lib():
    return L.load()


def _check(rc: int):
    if rc:
        msg = _lib().cheb_last_error().decode()
        raise _STATUS.get(rc, Error)(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _pd(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(L.F64P)


def _pi(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(L.I64P)


# ---------------------------------------------------------------------------
# coefficients.hpp:17-51
# ---------------------------------------------------------------------------


@dataclass
class CoefficientTable:
    c: float = 0.0
    beta: float = 0.0
    c0: float = 0.0
    coeffs: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class ApproxPlan:
    M: int = 0
    target_err: float = 0.0
    predicted_err: float = 0.0


def beta(c: float) -> float:
    o = C.c_double()
    _check(_lib().cheb_beta(c, C.byref(o)))
    return o.value


def sigma(c: float) -> float:
    o = C.c_double()
    _check(_lib().cheb_sigma(c, C.byref(o)))
    return o.value


def err_bound(c: float, M: int) -> float:
    o = C.c_double()
    _check(_lib().cheb_err_bound(c, M, C.byref(o)))
    return o.value


def plan_iterations(c: float, eps: float) -> ApproxPlan:
    M, p = C.c_int(), C.c_double()
    _check(_lib().cheb_plan_iterations(c, eps, C.byref(M), C.byref(p)))
    return ApproxPlan(M.value, eps, p.value)


def coefficients(c: float, M: int) -> CoefficientTable:
    out = np.zeros(max(M, 0) + 1)
    b, c0 = C.c_double(), C.c_double()
    _check(_lib().cheb_coefficients(c, M, _pd(out), C.byref(b), C.byref(c0)))
    return CoefficientTable(c, b.value, c0.value, out)


# ---------------------------------------------------------------------------
# graph.hpp:21-76
# ---------------------------------------------------------------------------


@dataclass
class UndirectedGraph:
    """Host CSR exactly as graph.hpp:21-31 (int64 arrays, fp64 inv_degree)."""
    n: int = 0
    m: int = 0
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.int64))
    neighbors: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    degrees: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    inv_degree: np.ndarray = field(default_factory=lambda: np.zeros(0))
    multi: bool = False

    def degree(self, v: int) -> int:
        return int(self.degrees[v])


@dataclass
class GraphStats:
    n: int = 0
    m: int = 0
    avg_degree: float = 0.0
    min_degree: int = 0
    max_degree: int = 0
    self_loops: int = 0
    duplicates_removed: int = 0
    isolated_dropped: int = 0


@dataclass
class BuildOptions:
    dedup: bool = True
    drop_isolated: bool = False
    n_hint: int = 0
    device: int = 0          # new
    row_ptr_64: bool = False  # new: int64 row pointers on the device


@dataclass
class BuildResult:
    graph: UndirectedGraph
    duplicates_removed: int = 0
    isolated_dropped: int = 0
    device_graph: Optional["DeviceGraph"] = None  # new: the resident device CSR


class DeviceGraph:
    """A device-resident graph handle (cheb_graph_t).  Owns GPU memory."""

    def __init__(self, handle: C.c_void_p, n: int):
        self._h = handle
        self.n = n

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = L.cheb_graph_info()
        _check(_lib().cheb_graph_get_info(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in L.cheb_graph_info._fields_}

    def download(self) -> UndirectedGraph:
        inf = self.info()
        n, nnz = inf["n"], inf["nnz"]
        off = np.zeros(n + 1, dtype=np.int64)
        nb = np.zeros(max(nnz, 1), dtype=np.int64)
        deg = np.zeros(max(n, 1), dtype=np.int64)
        _check(_lib().cheb_graph_download_csr(self._h, _pi(off), _pi(nb), _pi(deg)))
        deg = deg[:n]
        with np.errstate(divide="ignore"):
            inv = 1.0 / deg.astype(np.float64)
        return UndirectedGraph(n, inf["m"], off, nb[:nnz], deg, inv, bool(inf["multi"]))

    def free(self):
        if self._h:
            _lib().cheb_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.free()


def build_graph(edges, opts: Optional[BuildOptions] = None, keep_device: bool = False) -> BuildResult:
    """graph.hpp:60-61 — K1 device CSR builder; returns the host CSR like the reference."""
    opts = opts or BuildOptions()
    e = _i64(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    o = L.cheb_build_opts(int(opts.dedup), int(opts.drop_isolated), int(opts.n_hint),
                          int(opts.device), int(opts.row_ptr_64))
    h = C.c_void_p()
    inf = L.cheb_graph_info()
    _check(_lib().cheb_graph_build(_pi(e), e.shape[0], C.byref(o), C.byref(h), C.byref(inf)))
    dg = DeviceGraph(h, inf.n)
    g = dg.download()
    res = BuildResult(g, inf.duplicates_removed, inf.isolated_dropped)
    if keep_device:
        res.device_graph = dg
    else:
        dg.free()
    return res


def build_device_graph(edges, opts: Optional[BuildOptions] = None):
    """Build on the device and keep only the device handle (no host CSR download)."""
    opts = opts or BuildOptions()
    e = _i64(np.asarray(edges, dtype=np.int64).reshape(-1, 2))
    o = L.cheb_build_opts(int(opts.dedup), int(opts.drop_isolated), int(opts.n_hint),
                          int(opts.device), int(opts.row_ptr_64))
    h = C.c_void_p()
    inf = L.cheb_graph_info()
    _check(_lib().cheb_graph_build(_pi(e), e.shape[0], C.byref(o), C.byref(h), C.byref(inf)))
    return DeviceGraph(h, inf.n), {k: getattr(inf, k) for k, _ in L.cheb_graph_info._fields_}


@dataclass
class LoadOptions:
    """graph_io.hpp:24-28 (+ device placement)."""
    dedup: bool = True
    drop_isolated: bool = False
    symmetrize: bool = False
    device: int = 0          # new
    row_ptr_64: bool = False  # new


@dataclass
class LoadedGraph:
    """graph_io.hpp:30-33: the host CSR and its validated stats."""
    graph: UndirectedGraph
    stats: GraphStats
    device_graph: Optional["DeviceGraph"] = None  # new: the resident device CSR
    lines: int = 0                                # new: text lines consumed


def _load_opts(opts: Optional[LoadOptions]) -> "L.cheb_load_opts":
    opts = opts or LoadOptions()
    return L.cheb_load_opts(int(opts.dedup), int(opts.drop_isolated), int(opts.symmetrize),
                            int(opts.device), int(opts.row_ptr_64))


def _finish_load(rc: int, h: C.c_void_p, st, path: str, keep_device: bool) -> LoadedGraph:
    _check(rc)
    if st.weights_ignored:  # graph_io.cpp:134-138
        print(f"warning: {path}: real weights ignored, using pattern only", file=sys.stderr)
    if st.isolated_dropped > 0:  # graph_io.cpp:38-40
        print(f"warning: dropped {st.isolated_dropped} isolated vertices", file=sys.stderr)
    dg = DeviceGraph(h, st.n)
    stats = GraphStats(st.n, st.m, st.avg_degree, st.min_degree, st.max_degree, st.self_loops,
                       st.duplicates_removed, st.isolated_dropped)
    res = LoadedGraph(dg.download(), stats, None, st.lines)
    if keep_device:
        res.device_graph = dg
    else:
        dg.free()
    return res


def load_edge_list(path: str, opts: Optional[LoadOptions] = None, keep_device: bool = False) -> LoadedGraph:
    """graph_io.hpp:35 — the file is parsed on the GPU (line split + from_chars-exact ints)
    and built by K1; errors name the first failing line like graph_io.cpp:62-64."""
    h, st = C.c_void_p(), L.cheb_graph_stats()
    o = _load_opts(opts)
    rc = _lib().cheb_graph_load_edge_list(os.fsencode(path), C.byref(o), C.byref(h), C.byref(st))
    return _finish_load(rc, h, st, path, keep_device)


def load_matrix_market(path: str, opts: Optional[LoadOptions] = None, keep_device: bool = False) -> LoadedGraph:
    """graph_io.hpp:36 — header on the host, entries parsed and mirror-checked on the GPU."""
    h, st = C.c_void_p(), L.cheb_graph_stats()
    o = _load_opts(opts)
    rc = _lib().cheb_graph_load_matrix_market(os.fsencode(path), C.byref(o), C.byref(h), C.byref(st))
    return _finish_load(rc, h, st, path, keep_device)


def load_device_graph(path: str, fmt: str = "edges", opts: Optional[LoadOptions] = None):
    """Load straight to a resident device handle (no host CSR): (DeviceGraph, GraphStats)."""
    h, st = C.c_void_p(), L.cheb_graph_stats()
    o = _load_opts(opts)
    fn = _lib().cheb_graph_load_edge_list if fmt == "edges" else _lib().cheb_graph_load_matrix_market
    _check(fn(os.fsencode(path), C.byref(o), C.byref(h), C.byref(st)))
    return DeviceGraph(h, st.n), GraphStats(st.n, st.m, st.avg_degree, st.min_degree, st.max_degree,
                                            st.self_loops, st.duplicates_removed, st.isolated_dropped)


def parse_text(text: bytes, fmt: str = "edges", name: str = "<memory>",
               opts: Optional[LoadOptions] = None, keep_device: bool = False) -> LoadedGraph:
    """In-memory variant of the loaders (`name` stands in for the path in messages)."""
    h, st = C.c_void_p(), L.cheb_graph_stats()
    o = _load_opts(opts)
    rc = _lib().cheb_graph_parse_text(text, len(text), 0 if fmt == "edges" else 1, name.encode(),
                                      C.byref(o), C.byref(h), C.byref(st))
    return _finish_load(rc, h, st, name, keep_device)


def upload(g: UndirectedGraph, device: int = 0, row_ptr_64: bool = False) -> DeviceGraph:
    """Upload a host CSR (essential_check semantics, cpaa.cpp:16-26)."""
    off, nb, deg = _i64(g.offsets), _i64(g.neighbors), _i64(g.degrees)
    inv = _f64(g.inv_degree)
    if g.n < 1:
        raise ValidationError("graph has no vertices")
    h = C.c_void_p()
    _check(_lib().cheb_graph_upload_csr(_pi(off), off.size, _pi(nb), nb.size, _pi(deg), deg.size,
                                        _pd(inv), inv.size, int(g.n), int(g.m), int(g.multi),
                                        device, int(row_ptr_64), C.byref(h)))
    return DeviceGraph(h, g.n)


def _as_device(g, device: int = 0):
    """(DeviceGraph, owned?) for either a host UndirectedGraph or a DeviceGraph."""
    if isinstance(g, DeviceGraph):
        return g, False
    return upload(g, device), True


def transition_apply(g, x, mode: int = MODE_FAST) -> np.ndarray:
    """graph.hpp:64 — y = P x."""
    x = _f64(x)
    n = g.n
    if x.size != n:
        raise ValueError(f"vector length {x.size} does not match vertex count {n}")
    dg, owned = _as_device(g)
    try:
        y = np.zeros(n)
        _check(_lib().cheb_transition_apply(dg.handle, _pd(x), x.size, _pd(y), mode))
        return y
    finally:
        if owned:
            dg.free()


def kahan_sum(x) -> float:
    """graph.hpp:75-76 — compensated serial sum (host, graph.cpp:10-19)."""
    x = _f64(x)
    return _lib().cheb_kahan_sum(_pd(x), x.size)


def validate(g: UndirectedGraph, duplicates_removed: int = 0, isolated_dropped: int = 0) -> GraphStats:
    """graph.hpp:70-71 — structural re-check (graph.cpp:123-186) run on the device
    (cheb_validate_csr): the reference's check order and messages, first violation by vertex."""
    n = int(g.n)
    if n < 0:
        raise ValidationError("negative vertex count")
    off, nb, deg = _i64(g.offsets), _i64(g.neighbors), _i64(g.degrees)
    if off.size != n + 1:
        raise ValidationError("offsets length is not n+1")
    st = L.cheb_graph_stats()
    _check(_lib().cheb_validate_csr(_pi(off), off.size, _pi(nb), nb.size, _pi(deg), deg.size, n, int(g.m),
                                    int(bool(g.multi)), int(duplicates_removed), int(isolated_dropped), 0,
                                    C.byref(st)))
    return GraphStats(st.n, st.m, st.avg_degree, st.min_degree, st.max_degree, st.self_loops,
                      st.duplicates_removed, st.isolated_dropped)


# ---------------------------------------------------------------------------
# cpaa.hpp:27-85
# ---------------------------------------------------------------------------


@dataclass
class SolverConfig:
    c: float = 0.85
    rounds: int = -1
    eps: float = -1.0
    max_rounds: int = 60
    parallelism: int = 1
    # new, additive
    mode: int = MODE_FAST
    precision: int = 64
    personalization: Optional[np.ndarray] = None
    device: int = 0


@dataclass
class TraceRow:
    k: int = 0
    c_k: float = 0.0
    S_k: float = 0.0
    residual_mass: float = 0.0
    l1_change: float = 0.0
    elapsed_ms: float = 0.0
    mass_T: float = 0.0
    err: float = 0.0
    err_l1: float = 0.0


@dataclass
class PageRankResult:
    ranks: np.ndarray
    trace: list
    rounds: int = 0
    has_err: bool = False
    total_mass: float = 0.0


@dataclass
class VertexRange:
    begin: int = 0
    end: int = 0


def partition_vertices(g, K: int) -> list:
    """cpaa.hpp:66 — degree-balanced contiguous ranges (cpaa.cpp:40-68)."""
    deg = _i64(g.degrees) if not isinstance(g, DeviceGraph) else _i64(g.download().degrees)
    cuts = np.zeros(max(K, 0) + 1, dtype=np.int64)
    _check(_lib().cheb_partition_vertices(_pi(deg), deg.size, K, _pi(cuts)))
    return [VertexRange(int(cuts[j]), int(cuts[j + 1])) for j in range(K)]


def normalize(v) -> np.ndarray:
    """cpaa.hpp:69 — v / kahan_sum(v); NumericError unless the total is positive and finite."""
    v = _f64(v)
    total = kahan_sum(v)
    if not np.isfinite(total) or total <= 0.0:
        raise NumericError("normalization total is not positive and finite")
    return v / total


def _trace_rows(tr, M: int) -> list:
    return [TraceRow(r.k, r.c_k, r.S_k, r.residual_mass, r.l1_change, r.elapsed_ms, r.mass_T,
                     r.err, r.err_l1) for r in tr[:M]]


def _cpaa_opts(cfg: SolverConfig, p: Optional[np.ndarray]) -> L.cheb_cpaa_opts:
    o = L.cheb_cpaa_opts()
    _lib().cheb_cpaa_opts_default(C.byref(o))
    o.c, o.rounds, o.eps, o.max_rounds = cfg.c, cfg.rounds, cfg.eps, cfg.max_rounds
    o.parallelism, o.mode, o.precision = cfg.parallelism, cfg.mode, cfg.precision
    o.personalization = _pd(p)
    return o


def run_cpaa(g, cfg: Optional[SolverConfig] = None, reference=None) -> PageRankResult:
    """cpaa.hpp:74-75 — run_cpaa on the B200.

    ``g`` is a host UndirectedGraph (uploaded for this call, like the stateless
    reference API) or a resident DeviceGraph.
    """
    if isinstance(g, PartitionGroup):
        if reference is not None:
            raise ValueError("reference tracking is not available on a partitioned handle")
        return g.run_cpaa(cfg)
    cfg = cfg or SolverConfig()
    n = g.n
    if n < 1:
        raise ValidationError("graph has no vertices")
    dg, owned = _as_device(g, cfg.device)
    try:
        p = None if cfg.personalization is None else _f64(cfg.personalization)
        ref = None if reference is None else _f64(reference)
        o = _cpaa_opts(cfg, p)
        cap = max(cfg.max_rounds, cfg.rounds, 1) + 1
        tr = (L.cheb_trace_row * cap)()
        ranks = np.zeros(n)
        rounds, total = C.c_int(), C.c_double()
        _check(_lib().cheb_cpaa(dg.handle, C.byref(o), _pd(ref), 0 if ref is None else ref.size,
                                _pd(ranks), tr, C.byref(rounds), C.byref(total)))
        return PageRankResult(ranks, _trace_rows(tr, rounds.value), rounds.value,
                              ref is not None, total.value)
    finally:
        if owned:
            dg.free()


class PartitionGroup:
    """G row-partition ranks of one graph driven by this process (the fused push exchange,
    DESIGN.md §6): ``graphs[r]`` becomes rank r.  ``run_cpaa(group, cfg)`` solves over all
    ranks; on one GPU the ranks run in lockstep, on several they push x over peer memory."""

    def __init__(self, graphs: Sequence["DeviceGraph"]):
        self.graphs = list(graphs)
        arr = (C.c_void_p * len(self.graphs))(*[g.handle for g in self.graphs])
        self._h = C.c_void_p()
        _check(_lib().cheb_group_create(arr, len(self.graphs), C.byref(self._h)))
        self.n = self.graphs[0].n

    def run_cpaa(self, cfg: Optional[SolverConfig] = None) -> PageRankResult:
        cfg = cfg or SolverConfig()
        p = None if cfg.personalization is None else _f64(cfg.personalization)
        o = _cpaa_opts(cfg, p)
        cap = max(cfg.max_rounds, cfg.rounds, 1) + 1
        tr = (L.cheb_trace_row * cap)()
        ranks = np.zeros(self.n)
        rounds, total = C.c_int(), C.c_double()
        _check(_lib().cheb_group_cpaa(self._h, C.byref(o), _pd(ranks), tr, C.byref(rounds), C.byref(total)))
        return PageRankResult(ranks, _trace_rows(tr, rounds.value), rounds.value, False, total.value)

    def rank_term_ms(self, cfg: Optional[SolverConfig] = None) -> np.ndarray:
        """Mean term time of every rank's partition, the ranks' term kernels serialised so
        each is timed on the whole GPU (cheb_group_profile): the partition's load balance."""
        cfg = cfg or SolverConfig()
        o = _cpaa_opts(cfg, None)
        out = np.zeros(len(self.graphs))
        _check(_lib().cheb_group_profile(self._h, C.byref(o), _pd(out), out.size))
        return out

    def close(self):
        if self._h:
            _lib().cheb_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class BatchResult:
    ranks: np.ndarray        # n x R, column r normalised
    totals: np.ndarray       # R normalisation totals
    trace: list              # per term, sums over all R columns
    rounds: int = 0


def run_cpaa_batch(g, cfg: Optional[SolverConfig] = None, seeds=None, personalization=None) -> BatchResult:
    """Batched personalised CPAA (K5, config 5): one SpMM-shaped pass per term over R
    right-hand sides.  ``seeds`` (R vertex ids) gives one-hot columns; ``personalization``
    an explicit n x R block; neither = R=cfg-defined ones columns is not meaningful, so one
    of them is required."""
    cfg = cfg or SolverConfig()
    n = g.n
    if n < 1:
        raise ValidationError("graph has no vertices")
    sd = None if seeds is None else _i64(seeds)
    pp = None if personalization is None else _f64(personalization)
    if sd is None and pp is None:
        raise ValueError("give seeds or personalization")
    R = int(sd.size if sd is not None else pp.reshape(n, -1).shape[1])
    dg, owned = _as_device(g, cfg.device)
    try:
        o = _cpaa_opts(cfg, pp)
        o.R = R
        cap = max(cfg.max_rounds, cfg.rounds, 1) + 1
        tr = (L.cheb_trace_row * cap)()
        ranks = np.zeros(n * R)
        totals = np.zeros(R)
        rounds = C.c_int()
        _check(_lib().cheb_cpaa_batch(dg.handle, C.byref(o), _pi(sd), _pd(ranks), _pd(totals), tr,
                                      C.byref(rounds)))
        return BatchResult(ranks.reshape(n, R), totals, _trace_rows(tr, rounds.value), rounds.value)
    finally:
        if owned:
            dg.free()


class IterationState:
    """cpaa.hpp:79-82 — staged state, device-backed (same arithmetic as run_cpaa)."""

    def __init__(self, dg: DeviceGraph, owned: bool, mode: int):
        self._dg, self._owned, self.mode = dg, owned, mode

    def _get(self):
        n = self._dg.n
        a = [np.zeros(n) for _ in range(4)]
        k = C.c_int()
        _check(_lib().cheb_state_get(self._dg.handle, *[_pd(x) for x in a], C.byref(k)))
        return a, k.value

    @property
    def T_prev(self):
        return self._get()[0][0]

    @property
    def T_curr(self):
        return self._get()[0][1]

    @property
    def T_next(self):
        return self._get()[0][2]

    @property
    def acc(self):
        return self._get()[0][3]

    @property
    def k(self):
        return self._get()[1]

    def set(self, T_prev=None, T_curr=None, acc=None, k: int = 0):
        tp = None if T_prev is None else _f64(T_prev)
        tc = None if T_curr is None else _f64(T_curr)
        ac = None if acc is None else _f64(acc)
        _check(_lib().cheb_state_set(self._dg.handle, _pd(tp), _pd(tc), _pd(ac), k))

    def rotate(self):
        """T_prev <- T_curr <- T_next; k += 1 (the caller's swaps in test_cpaa.cpp:163-166)."""
        _check(_lib().cheb_state_rotate(self._dg.handle))

    def close(self):
        if self._owned:
            self._dg.free()


def init_state(g, c0: float, mode: int = MODE_FAST) -> IterationState:
    """cpaa.hpp:83 init_state."""
    if g.n < 1:
        raise ValidationError("graph has no vertices")
    dg, owned = _as_device(g)
    _check(_lib().cheb_state_init(dg.handle, c0, mode))
    return IterationState(dg, owned, mode)


def generate_stage(state: IterationState) -> None:
    """cpaa.hpp:84 generate_stage (the graph is the state's)."""
    _check(_lib().cheb_state_generate(state._dg.handle))


def accumulate_stage(state: IterationState, c_k: float) -> None:
    """cpaa.hpp:85 accumulate_stage."""
    _check(_lib().cheb_state_accumulate(state._dg.handle, c_k))


# ---------------------------------------------------------------------------
# power.hpp:13-28
# ---------------------------------------------------------------------------


@dataclass
class PowerConfig:
    c: float = 0.85
    rounds: int = -1
    tol: float = -1.0
    max_rounds: int = 60
    parallelism: int = 1
    mode: int = MODE_FAST
    device: int = 0


def run_power(g, cfg: Optional[PowerConfig] = None, reference=None) -> PageRankResult:
    """power.hpp:24-25 — the Power-method comparator on the B200."""
    cfg = cfg or PowerConfig()
    n = g.n
    if n < 1:
        raise ValidationError("graph has no vertices")
    dg, owned = _as_device(g, cfg.device)
    try:
        ref = None if reference is None else _f64(reference)
        o = L.cheb_power_opts(cfg.c, cfg.rounds, cfg.tol, cfg.max_rounds, cfg.parallelism, cfg.mode)
        cap = max(cfg.rounds if cfg.rounds >= 0 else cfg.max_rounds, 1)
        tr = (L.cheb_trace_row * cap)()
        ranks = np.zeros(n)
        rounds, total = C.c_int(), C.c_double()
        _check(_lib().cheb_power(dg.handle, C.byref(o), _pd(ref), 0 if ref is None else ref.size,
                                 _pd(ranks), tr, cap, C.byref(rounds), C.byref(total)))
        return PageRankResult(ranks, _trace_rows(tr, rounds.value), rounds.value,
                              ref is not None, total.value)
    finally:
        if owned:
            dg.free()


def reference_pagerank(g, c: float, mode: int = MODE_FAST) -> np.ndarray:
    """power.hpp:28 — the 210-round reference vector."""
    return run_power(g, PowerConfig(c=c, rounds=210, parallelism=1, mode=mode)).ranks


def device_count() -> int:
    return _lib().cheb_device_count()

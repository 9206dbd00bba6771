#!/usr/bin/env python
"""Benchmark of the CPAA hot path (BASELINE.json metric: GTEPS per Chebyshev term and
time-to-1e-10 on B200, with the HBM-roofline fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--precision 64]
    python bench.py --impl reference ...      # the reference's own CPU run_cpaa

A step = one full CPAA solve to L1 error 1e-10 (M = plan_iterations(0.85, 1e-10) = 39
fused terms + normalisation) over the configuration's synthetic graph, graph resident in
HBM.  value = whole-job GTEPS = nnz * M / step_time (every CSR entry is one traversal).
L2 is flushed (a 512 MiB write) before every timed step; the flush is outside the
timed events.  e2e = the same metric through the reference-facing C-ABI call with HOST
buffers (CSR upload from pinned memory + solve + ranks read-back, every step).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EPS = 1e-10
DAMPING = 0.85

# BASELINE.json configs (synthetic stand-ins; seeds fixed here).
CONFIGS = {
    "c1": dict(kind="gnp", n=10_000, p=0.001, seed=1, drop=False,
               desc="gnp(10000, 0.001, seed 1), config 1 (CPU parity config)"),
    "c2": dict(kind="chung_lu", n=1 << 20, gamma=2.1, wmin=2.0, wmax=50_000.0,
               draws=10_485_760, seed=2, drop=False,
               desc="Chung-Lu n=2^20, exponent 2.1, weights [2,50000], ~10M undirected edges"),
    "c3": dict(kind="rmat", scale=22, ef=16, seed=3, drop=True,
               desc="R-MAT scale 22, ef 16, (0.57,0.19,0.19,0.05), relabelled, isolated dropped"),
    "c4": dict(kind="rmat", scale=25, ef=16, seed=4, drop=True, rp64=True,
               desc="R-MAT scale 25, ef 16, int64 row pointers, isolated dropped"),
    "c5": dict(kind="chung_lu", n=1 << 22, gamma=2.1, wmin=2.0, wmax=50_000.0,
               draws=41_943_040, seed=5, drop=False, R=64,
               desc="Chung-Lu n=2^22, ~40M undirected edges, 64 one-hot seeds (degree >= 5), SpMM R=64"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------------------
# distributed plumbing (torch.distributed only for barrier / max-over-ranks)
# ----------------------------------------------------------------------------------------
class Dist:
    def __init__(self, n_gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            import torch
            self.pg.barrier()
            torch.cuda.synchronize()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{self.local}")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def min(self, x: float) -> float:
        return -self.max(-x)

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------------------
# clocks sampling during the timed region
# ----------------------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler (5 ms period) started before the timed region; summary() keeps the
    samples whose arrival time falls inside [mark_start, mark_end] (+ one period of slack)."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.samples = []  # (host time, line)
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "5"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 3.0
            while not self.samples and time.time() < deadline:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(0.02)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo = (self.t0 or 0) - 0.006
        hi = (self.t1 or time.time()) + 0.006
        window = [ln for t, ln in self.samples if lo <= t <= hi]
        for ln in window:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "period_ms": 5}


# ----------------------------------------------------------------------------------------
# inputs
# ----------------------------------------------------------------------------------------
def config_dict(name: str, n: int, nnz: int, M: int, R: int) -> dict:
    """The workload as both arms name it (identical dicts: same graph, terms, c, eps)."""
    return {"workload": name, "desc": CONFIGS[name]["desc"], "n": n, "nnz": nnz, "R": R, "terms": M,
            "eps": EPS, "c": DAMPING, "seed": CONFIGS[name]["seed"],
            "l2": "GPU arm: flushed (512 MiB write) before every timed step"}


def make_edges_device(cfg: dict, device: int):
    """GPU arm: the product generators (counter-based R-MAT / Chung-Lu on the device)."""
    from paper_2112_01743_b200 import generate as G
    if cfg["kind"] == "gnp":
        return G.gnp_edges(cfg["n"], cfg["p"], cfg["seed"])
    if cfg["kind"] == "chung_lu":
        return G.chung_lu_edges(cfg["n"], cfg["gamma"], cfg["wmin"], cfg["wmax"], cfg["draws"],
                                cfg["seed"], device=device)
    return G.rmat_edges(cfg["scale"], cfg["ef"], 0.57, 0.19, 0.19, cfg["seed"], device=device)


def make_edges_host(cfg: dict) -> np.ndarray:
    """CPU legs: the same edge list without the product library — the reference's own gnp
    generator (config 1) or the plain-C restatement of the config generators
    (oracle/synth_gen.c, pinned equal to the product's by tests/test_oracle.py)."""
    from oracle import Oracle, Reference
    if cfg["kind"] == "gnp":
        return Reference().gnp_edges(cfg["n"], cfg["p"], cfg["seed"])
    o = Oracle()
    if cfg["kind"] == "chung_lu":
        return o.chung_lu_edges(cfg["n"], cfg["gamma"], cfg["wmin"], cfg["wmax"], cfg["draws"], cfg["seed"])
    return o.rmat_edges(cfg["scale"], cfg["ef"], 0.57, 0.19, 0.19, cfg["seed"])


def build_device(cfg: dict, device: int):
    """Generate on the device and run the K1 builder there (no host round trip)."""
    import paper_2112_01743_b200 as cheb
    from paper_2112_01743_b200 import _lib as L
    lib = L.load()
    e = make_edges_device(cfg, device)
    o = L.cheb_build_opts(1, int(cfg.get("drop", False)), 0, device, int(cfg.get("rp64", False)))
    h = C.c_void_p()
    inf = L.cheb_graph_info()
    if isinstance(e, np.ndarray):
        e64 = np.ascontiguousarray(e.astype(np.int64))
        rc = lib.cheb_graph_build(e64.ctypes.data_as(L.I64P), e64.shape[0], C.byref(o), C.byref(h), C.byref(inf))
        E = e64.shape[0]
    else:
        rc = lib.cheb_graph_build_device(C.c_void_p(e.ptr), e.count, 32, C.byref(o), C.byref(h), C.byref(inf))
        E = e.count
        e.free()
    cheb.api._check(rc)
    info = {k: getattr(inf, k) for k, _ in L.cheb_graph_info._fields_}
    info["edges_drawn"] = E
    return cheb.DeviceGraph(h, inf.n), info


def algorithmic_bytes(n: int, nnz: int, rp_bytes: int, vbytes: int, R: int = 1) -> int:
    """B_term = 4 nnz + I_r (n+1) + 6 V R n."""
    return 4 * nnz + rp_bytes * (n + 1) + 6 * vbytes * R * n


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------------------
# CPU legs: the reference compiled unmodified (oracle/_ref), or the restated loop (R > 1)
# ----------------------------------------------------------------------------------------
CPU_STEP_TARGET_S = 6.0   # one reference step is a bounded sample of the workload


def _rounds_for(t_round_ms: float, M: int, target_s: float) -> int:
    return int(min(M, max(1, math.ceil(target_s * 1e3 / max(t_round_ms, 1e-3)))))


def ref_sample(rg, M: int, threads: int, target_s: float):
    """Calibrate with a 1-round run, then size the sample (rounds <= M) to ~target_s."""
    t1 = rg.run_cpaa(c=DAMPING, rounds=1, parallelism=threads).wall_ms
    return _rounds_for(t1, M, target_s)


def port_columns(csr, seeds, M: int, rounds: int, threads: int):
    """The restated loop (oracle/cpaa_oracle.c, cpaa.cpp:79-165 with T0 = e_seed) for
    `threads` one-hot columns at once, one host thread each (ctypes drops the GIL).
    Returns (wall_ms, columns)."""
    from oracle import Oracle
    o = Oracle()
    cols = [int(s) for s in seeds[:threads]]

    def one(s):
        p = np.zeros(csr.n)
        p[s] = 1.0
        o.run_cpaa(csr, rounds, p=p)
    ths = [threading.Thread(target=one, args=(s,)) for s in cols]
    t = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return (time.perf_counter() - t) * 1e3, len(cols)


def c5_seeds_from_degrees(deg, R: int, seed: int = 5):
    """R seed vertices drawn uniformly (without replacement) from vertices of degree >= 5,
    with a fixed counter-based draw (splitmix64), so both arms use the same seeds."""
    cand = np.nonzero(np.asarray(deg) >= 5)[0]
    out, used, i = [], set(), 0
    M64 = (1 << 64) - 1
    while len(out) < R:
        z = (seed * 0x9E3779B97F4A7C15 + i * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        z ^= z >> 31
        v = int(cand[z % len(cand)])
        i += 1
        if v not in used:
            used.add(v)
            out.append(v)
    return np.array(out, dtype=np.int64)


def run_reference_arm(args):
    """--impl reference: the reference's own CPU run_cpaa (oracle/_ref = the unmodified
    sources) on this box's host cores, on the same graph (edges from oracle/synth_gen.c; the
    product library is never loaded).  One step = one run_cpaa call with a bounded round
    count (calibrated to ~6 s; all M = 39 rounds when that fits); value = nnz * rounds /
    wall.  For the batched config the reference has no personalisation: the restated loop
    (oracle/cpaa_oracle.c) over one-hot columns, one host thread per column."""
    cfgname = args.config
    cfg = CONFIGS[cfgname]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    try:
        from oracle import REF_SO, Reference
        if not os.path.exists(REF_SO):
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return 0
        threads = host_threads()
        ref = Reference()
        t0 = time.perf_counter()
        e = make_edges_host(cfg)
        gen_s = time.perf_counter() - t0
        E = int(e.shape[0])
        t0 = time.perf_counter()
        rg = ref.build_graph(e, dedup=True, drop_isolated=cfg.get("drop", False))
        build_s = time.perf_counter() - t0
        del e
        M, _ = ref.plan_iterations(DAMPING, EPS)
        R = int(cfg.get("R", 1))
        walls = []
        if R > 1:
            csr = rg.csr()
            seeds = c5_seeds_from_degrees(csr.degrees, R)
            w1, _ = port_columns(csr, seeds, M, 1, threads)
            rounds = _rounds_for(w1, M, CPU_STEP_TARGET_S)
            for i in range(args.warmup + args.steps):
                w, cols = port_columns(csr, seeds, M, rounds, threads)
                if i >= args.warmup:
                    walls.append(w)
            units = rg.nnz * cols * rounds
            kind, what = "port", (f"restated loop (oracle/cpaa_oracle.c, T0 = e_seed) on {cols} of the {R} "
                                  f"one-hot columns at once, {rounds} rounds each, one host thread per column; "
                                  f"unit nnz*columns*rounds / wall (the reference has no personalisation)")
        else:
            rounds = ref_sample(rg, M, threads, CPU_STEP_TARGET_S)
            for i in range(args.warmup + args.steps):
                r = rg.run_cpaa(c=DAMPING, rounds=rounds, parallelism=threads)
                if i >= args.warmup:
                    walls.append(r.wall_ms)
            units = rg.nnz * rounds
            kind, what = "reference", (f"run_cpaa(c=0.85, rounds={rounds} of the M={M} terms to eps 1e-10, "
                                       f"parallelism={threads}) per step, steady_clock wall around the call")
    except Exception as ex:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"{type(ex).__name__}: {ex}"}))
        return 0
    ms = statistics.mean(walls)
    gteps = units / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference",
        "metric": "cpaa_gteps_per_term",
        "value": round(gteps, 6),
        "unit": "GTEPS",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(cfgname, rg.n, rg.nnz, M, R),
        "parallelism": f"cpu{threads}",
        "cpu_baseline": {"value": round(gteps, 6), "unit": "GTEPS", "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{cfgname}: {what}; edges generated in {gen_s:.1f}s ({E} pairs), "
                                   f"reference build_graph {build_s:.1f}s (excluded)"},
        "e2e": {"value": round(gteps, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline_line(solver, cfgname, args):
    """The reference compiled unmodified (oracle/_ref) timed on this box's host cores on the
    SAME CSR (downloaded; bit-exact with the reference's build_graph by the parity tests, so
    no rebuild): a bounded sample at K = every host thread and at K = 1.  For the batched
    config: the restated loop over one-hot columns (one host thread per column)."""
    try:
        from oracle import CSR, Reference
        host = solver.dg.download()
        threads = host_threads()
        M = solver.M
        csr = CSR(host.n, host.m, host.offsets, host.neighbors, host.degrees, host.inv_degree)
        if solver.R > 1:
            w1, _ = port_columns(csr, solver.seeds_all, M, 1, threads)
            rounds = _rounds_for(w1, M, CPU_STEP_TARGET_S)
            w, cols = port_columns(csr, solver.seeds_all, M, rounds, threads)
            wk1, _ = port_columns(csr, solver.seeds_all, M, 1, 1)
            v = host.neighbors.size * cols * rounds / (w * 1e-3) / 1e9
            v1 = host.neighbors.size * 1 * 1 / (wk1 * 1e-3) / 1e9
            return {"value": round(v, 6), "unit": "GTEPS", "cores": threads, "kind": "port",
                    "cpu_model": cpu_model(),
                    "k1": {"value": round(v1, 6), "cores": 1, "sample": f"1 column, 1 round, wall {wk1:.0f} ms"},
                    "sample": f"restated loop (oracle/cpaa_oracle.c, T0 = e_seed), {cols} one-hot columns at once "
                              f"x {rounds} rounds, one host thread per column, wall {w:.0f} ms; unit nnz*columns*rounds"}
        rg = Reference().graph_from_csr(csr)
        del host
        rk = ref_sample(rg, M, threads, CPU_STEP_TARGET_S)
        wk = rg.run_cpaa(c=DAMPING, rounds=rk, parallelism=threads).wall_ms
        t1 = rg.run_cpaa(c=DAMPING, rounds=1, parallelism=1).wall_ms
        r1 = _rounds_for(t1, M, CPU_STEP_TARGET_S / 2)
        w1 = rg.run_cpaa(c=DAMPING, rounds=r1, parallelism=1).wall_ms if r1 > 1 else t1
        nnz = rg.nnz
        return {"value": round(nnz * rk / (wk * 1e-3) / 1e9, 6), "unit": "GTEPS", "cores": threads,
                "kind": "reference", "cpu_model": cpu_model(),
                "k1": {"value": round(nnz * r1 / (w1 * 1e-3) / 1e9, 6), "cores": 1,
                       "sample": f"run_cpaa(rounds={r1}, parallelism=1), wall {w1:.0f} ms"},
                "sample": f"run_cpaa(rounds={rk} of M={M}, parallelism={threads}) on the same {cfgname} CSR "
                          f"({nnz} entries), wall {wk:.0f} ms; build excluded"}
    except Exception as ex:  # noqa: BLE001
        return {"value": None, "unit": "GTEPS", "cores": 0, "kind": "reference",
                "sample": f"failed: {type(ex).__name__}: {ex}"}


# ----------------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------------
class _Handle:
    def __init__(self, h):
        self.handle = h


class Solver:
    """One step = one CPAA solve to eps 1e-10 on the resident graph (scalar K2 path, or the
    batched K5 path when the config has R right-hand sides)."""

    def __init__(self, dg, info, cfg, precision, rank=0, world=1):
        import paper_2112_01743_b200 as cheb
        from paper_2112_01743_b200 import _lib as L
        self.cheb, self.L, self.lib = cheb, L, L.load()
        self.dg, self.info, self.cfg = dg, info, cfg
        self.R = int(cfg.get("R", 1))
        self.M = cheb.plan_iterations(DAMPING, EPS).M
        self.seeds_all = None
        self.seeds = None
        if self.R > 1:
            self.seeds_all = c5_seeds_from_degrees(np.diff(dg.download().offsets), self.R)
            self.seeds = self.seeds_all
            if world > 1:
                # batched config on N GPUs: replicas (§8(e)) — the graph on every GPU, the R
                # right-hand sides split across the ranks, no per-term communication
                self.seeds = np.ascontiguousarray(self.seeds_all[rank::world])
                self.R = int(self.seeds.size)
        o = L.cheb_cpaa_opts()
        self.lib.cheb_cpaa_opts_default(C.byref(o))
        o.eps, o.c, o.precision, o.R = EPS, DAMPING, precision, self.R
        self.opts = o
        o0 = L.cheb_cpaa_opts()
        self.lib.cheb_cpaa_opts_default(C.byref(o0))
        o0.eps, o0.rounds, o0.c, o0.precision, o0.R = -1.0, 0, DAMPING, precision, self.R
        self.opts0 = o0  # the same solve with zero terms (init + normalise only)
        self.d_ranks = C.c_void_p()

    def _seed_ptr(self):
        return None if self.seeds is None else self.seeds.ctypes.data_as(self.L.I64P)

    def solve(self, handle=None, zero_terms=False):
        h = handle or self.dg.handle
        o = self.opts0 if zero_terms else self.opts
        if self.R > 1:
            self.cheb.api._check(self.lib.cheb_cpaa_batch(h, C.byref(o), self._seed_ptr(),
                                                          None, None, None, None))
        else:
            self.cheb.api._check(self.lib.cheb_cpaa_device(h, C.byref(o), C.byref(self.d_ranks), 0))

    def last_ms(self):
        lm, tm, terms, launches = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        self.cheb.api._check(self.lib.cheb_last_timing(self.dg.handle, C.byref(lm), C.byref(tm),
                                                       C.byref(terms), C.byref(launches)))
        return lm.value, launches.value

    def term_us_replayed(self, flush, reps):
        """Average duration of one term (term kernel + hub finalize + its share of the trace
        reduction) in the SAME graph-replayed, PDL-chained solve the timed step runs:
        (t(M terms) - t(0 terms)) / M, each the mean of `reps` graph replays with L2 flushed
        (CUDA events on the library's stream)."""
        import torch

        def mean_ms(zero):
            for _ in range(3):  # first: plain launches; second: capture; then replays
                self.solve(zero_terms=zero)
                self.last_ms()
            ts = []
            for _ in range(reps):
                flush.zero_()
                torch.cuda.synchronize()
                self.solve(zero_terms=zero)
                ts.append(self.last_ms()[0])
            return statistics.mean(ts)
        t0 = mean_ms(True)
        tM = mean_ms(False)
        return (tM - t0) / self.M * 1e3, tM, t0

    def e2e(self, device, steps, flush, dist, exchange, warmup=3):
        """Through the reference-facing C-ABI with host buffers: pinned int64 CSR upload,
        solve, ranks (and trace) read back to host memory, every step.  N > 1: every step's
        fresh handle joins the row-partitioned solve with the same exchange as the timed
        loop (fused push: IPC-mapped peer buffers; or an NCCL communicator)."""
        import torch
        L, lib = self.L, self.lib
        host = self.dg.download()
        n, R = host.n, self.R
        off = torch.from_numpy(host.offsets).pin_memory().numpy()
        nb = torch.from_numpy(host.neighbors).pin_memory().numpy()
        deg = host.degrees  # read on the host only (essential checks)
        inv = torch.from_numpy(host.inv_degree).pin_memory().numpy()
        ranks = torch.empty(n * R, dtype=torch.float64).pin_memory().numpy()
        tr = (L.cheb_trace_row * 64)()
        rounds, tot = C.c_int(), C.c_double()
        totals = np.zeros(R)
        comm = None
        if dist.world > 1 and self.R_cfg == 1 and exchange == "nccl":
            from paper_2112_01743_b200.distributed import Communicator
            comm = Communicator(dist.rank, dist.world, device)

        def step():
            h = C.c_void_p()
            self.cheb.api._check(lib.cheb_graph_upload_csr(
                off.ctypes.data_as(L.I64P), off.size, nb.ctypes.data_as(L.I64P), nb.size,
                deg.ctypes.data_as(L.I64P), deg.size, inv.ctypes.data_as(L.F64P), inv.size,
                n, int(host.m), 0, device, int(self.info["row_ptr_64"]), C.byref(h)))
            px = None
            if dist.world > 1 and self.R_cfg == 1:
                if comm is not None:
                    self.cheb.api._check(lib.cheb_graph_attach_comm(h, comm.handle))
                else:
                    from paper_2112_01743_b200.distributed import PeerExchange
                    px = PeerExchange(_Handle(h), dist.rank, dist.world)
            if R > 1:
                self.cheb.api._check(lib.cheb_cpaa_batch(h, C.byref(self.opts), self._seed_ptr(),
                                                         ranks.ctypes.data_as(L.F64P),
                                                         totals.ctypes.data_as(L.F64P), tr, C.byref(rounds)))
            else:
                self.cheb.api._check(lib.cheb_cpaa(h, C.byref(self.opts), None, 0, ranks.ctypes.data_as(L.F64P),
                                                   tr, C.byref(rounds), C.byref(tot)))
            if px is not None:
                px.detach()
            lib.cheb_graph_free(h)

        if dist.world > 1 and self.R_cfg == 1 and comm is None:
            # push exchange on fresh handles: every rank must map its peers; if any rank
            # cannot, every rank switches the e2e leg to the NCCL exchange together
            err = None
            try:
                step()
            except Exception as ex:  # noqa: BLE001
                err = f"{type(ex).__name__}: {str(ex)[:120]}"
            if dist.min(0.0 if err else 1.0) < 1.0:
                log(f"e2e: push exchange unavailable ({err or 'on a peer rank'}); NCCL all-gather")
                from paper_2112_01743_b200.distributed import Communicator
                comm = Communicator(dist.rank, dist.world, device)
        # pool, pinned staging and page-cache warm-up: the memory pool can take a few uploads to
        # settle on a fresh box (cudaMallocAsync of the 4 GB view buffers: 0.2-0.9 s instead of
        # microseconds, tools/e2e_breakdown.py with CHEB_DEBUG_ALLOC=1)
        for _ in range(max(5, warmup)):
            step()
        dist.barrier()
        times = []
        for _ in range(max(1, steps)):
            flush.zero_()
            torch.cuda.synchronize()
            t = time.perf_counter()
            step()
            times.append(time.perf_counter() - t)
        if comm is not None:
            comm.close()
        if os.environ.get("CHEB_BENCH_VERBOSE"):
            log("e2e steps (ms): " + " ".join(f"{1e3 * t:.2f}" for t in times))
        e2e_s = dist.max(statistics.mean(times))
        units = self.info["nnz"] * self.R_cfg * self.M
        exch = ("" if dist.world == 1 or self.R_cfg > 1 else
                (" + NCCL communicator" if comm is not None else " + push exchange (IPC peer mapping)"))
        return {"value": round(units / e2e_s / 1e9, 4), "unit": "GTEPS",
                # inv_degree is checked bitwise on the host threads and, being canonical,
                # never copied (a non-canonical one would add n * 8 bytes)
                "h2d_bytes_per_step": int(off.nbytes + nb.nbytes),
                "d2h_bytes_per_step": int(ranks.nbytes + 2 * self.M * 8),
                "ms_per_step": round(e2e_s * 1e3, 3),
                "path": "cheb_graph_upload_csr(pinned int64 CSR; inv_degree verified on the host)" + exch + " + " +
                        ("cheb_cpaa_batch" if R > 1 else "cheb_cpaa") + "(host ranks) + cheb_graph_free"}


def lsu_roofline(config, precision, world, mean_launch_us, sm_mhz):
    """Second roofline for the gather-bound term kernel: L1TEX data-pipe wavefronts per
    launch (ncu, profiles/traffic.json) over one wavefront per cycle per SM."""
    if world != 1 or not sm_mhz:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            w = json.load(f).get(f"{config}/f{precision}", {}).get("lsu_wavefronts")
    except (OSError, ValueError):
        return None
    if not w:
        return None
    peak = 148 * sm_mhz * 1e6  # wavefronts / s
    floor_us = w / peak * 1e6
    return {"bound": "l1tex_lsu_wavefronts", "wavefronts_per_launch": w, "peak_wavefronts_per_s": round(peak),
            "floor_us": round(floor_us, 1), "achieved_us": round(mean_launch_us, 1),
            "frac": round(floor_us / mean_launch_us, 4),
            "source": "wavefronts from the committed ncu capture (profiles/traffic.json)"}


def window_info(dg):
    """The resident view's column windows (hub-row entries gathered from shared memory by
    k_window_pass), or None when the view has none."""
    from paper_2112_01743_b200 import _lib as L
    sizes = np.zeros(8, dtype=np.int64)
    if L.load().cheb_graph_view_windows(dg.handle, sizes.ctypes.data_as(L.I64P), None, None, None, None, None) != 0:
        return None
    if sizes[0] <= 0:
        return None
    return {"windows": int(sizes[0]), "ids_per_window": int(sizes[1]), "first_id": int(sizes[2]),
            "entries": int(sizes[4]), "piece_sums": int(sizes[5]), "chunk_tiles_left": int(sizes[6])}


def measured_traffic(config, precision, world):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/traffic.json), or None when this workload has not been captured."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(f"{config}/f{precision}", {}).get("bytes")
    except (OSError, ValueError):
        return None


def power_comparator(dg, flush, precision):
    """The paper's comparison on the same resident graph: CPAA to L1 error 1e-10 (39 terms)
    against the Power method for its a-priori round count 2 c^k <= 1e-10 (146 rounds),
    both through the public API with the ranks read back (wall clock, L2 flushed, best of 3)."""
    import torch
    import paper_2112_01743_b200 as cheb
    k_pow = 1
    while 2.0 * DAMPING ** k_pow > EPS:
        k_pow += 1

    def best(fn):
        fn()
        ts = []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t)
        return min(ts) * 1e3
    p_ms = best(lambda: cheb.run_power(dg, cheb.PowerConfig(c=DAMPING, rounds=k_pow)))
    c_ms = best(lambda: cheb.run_cpaa(dg, cheb.SolverConfig(c=DAMPING, eps=EPS, precision=precision)))
    return {"cpaa_api_ms": round(c_ms, 3), "cpaa_terms": cheb.plan_iterations(DAMPING, EPS).M,
            "power_api_ms": round(p_ms, 3), "power_rounds": k_pow, "power_dtype": "f64",
            "speedup": round(p_ms / c_ms, 2),
            "note": "same resident graph, public API incl. ranks read-back, wall clock, best of 3"}


def timed_steps(sv, flush, steps, dist, clk=None):
    """Time exactly `steps` solves (CUDA events on the library's stream, L2 flushed before
    each, outside the events); returns (ms_per_step max over ranks, our kernel launches)."""
    import torch
    dist.barrier()
    torch.cuda.synchronize()
    times, launches = [], 0
    if clk:
        clk.mark_start()
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        sv.solve()
        ms, nl = sv.last_ms()
        times.append(ms)
        launches += nl
    torch.cuda.synchronize()
    if clk:
        clk.mark_end()
    dist.barrier()
    return dist.max(sum(times)) / steps, launches


def secondary_line(name, device, precision, steps, warmup, dist):
    """A compact measurement of a second workload (C2 next to the C4 headline; "c4:32" = the
    headline graph in fp32)."""
    import torch
    if ":" in name:
        name, p = name.split(":")
        precision = int(p)
    cfg = CONFIGS[name]
    dg, info = build_device(cfg, device)
    sv = Solver(dg, info, cfg, precision)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    for _ in range(warmup):
        sv.solve()
        sv.last_ms()
    ms, _ = timed_steps(sv, flush, steps, dist)
    term_us, _, _ = sv.term_us_replayed(flush, max(3, steps // 2))
    n, nnz = info["n"], info["nnz"]
    B = algorithmic_bytes(n, nnz, 8 if info["row_ptr_64"] else 4, 8 if precision == 64 else 4, sv.R)
    peak, _ = peaks()
    ach = B / (term_us * 1e-6) / 1e9
    dg.free()
    return {"config": config_dict(name, n, nnz, sv.M, sv.R), "value": round(nnz * sv.R * sv.M / (ms * 1e-3) / 1e9, 3),
            "unit": "GTEPS", "dtype": "f64" if precision == 64 else "f32", "ms_per_step": round(ms, 4), "steps": steps,
            "roofline": {"achieved": round(ach, 1), "peak": peak, "frac": round(ach / peak, 4),
                         "mean_launch_us": round(term_us, 3), "bytes_per_launch": B}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS),
                    help="workload (default c4: the largest single-GPU config, the scaling graph)")
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--secondary", default="c2,c4:32",
                    help="comma list of extra workloads measured compactly at N=1, name[:precision] ('' for none)")
    ap.add_argument("--exchange", default="push", choices=["push", "nccl"],
                    help="N>1: x_{k+1} exchange of the row partition (fused push over peer memory, "
                         "or NCCL all-gather); the e2e leg uses the same exchange")
    ap.add_argument("--profile-only", action="store_true",
                    help="build + a few solves, no timing output (for ncu captures)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile_only else args.warmup

    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    dist = Dist(args.gpus)
    device = dist.local
    torch.cuda.set_device(device)
    cfg = CONFIGS[args.config]

    t0 = time.perf_counter()
    dg, info = build_device(cfg, device)
    build_s = time.perf_counter() - t0
    comm = px = None
    exchange_note = None
    R_cfg = int(cfg.get("R", 1))
    exchange = args.exchange
    if dist.world > 1 and R_cfg == 1:
        # strong scaling: every rank holds the same graph; the solver view is partitioned by
        # rows over the ranks and x_{k+1} reaches every rank each term — pushed by the term
        # kernels into the peers' buffers (default) or all-gathered by NCCL
        from paper_2112_01743_b200.distributed import Communicator, PeerExchange
        if exchange == "push":
            err = None
            try:
                px = PeerExchange(dg, dist.rank, dist.world)
                Solver(dg, info, cfg, args.precision, dist.rank, dist.world).solve()  # barrier works?
            except Exception as ex:  # noqa: BLE001 — no peer mapping: the NCCL baseline exchange
                err = f"{type(ex).__name__}: {str(ex)[:120]}"
            if dist.min(0.0 if err else 1.0) < 1.0:  # every rank takes the same exchange
                exchange_note = f"push unavailable ({err or 'on a peer rank'}); nccl all-gather"
                log(exchange_note)
                if px is not None:
                    px.detach()
                px = None
                exchange = "nccl"
        if exchange == "nccl":
            comm = Communicator(dist.rank, dist.world, device)
            comm.attach(dg)
    n, nnz = info["n"], info["nnz"]
    sv = Solver(dg, info, cfg, args.precision, dist.rank, dist.world)
    sv.R_cfg = R_cfg
    M, R = sv.M, sv.R

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    for _ in range(args.warmup):
        sv.solve()
        sv.last_ms()
    if args.profile_only:
        torch.cuda.synchronize()
        log(f"profile-only: n={n} nnz={nnz} R={R} built in {build_s:.2f}s")
        return 0

    with Clocks(device) as clk:
        ms_step, launches = timed_steps(sv, flush, args.steps, dist, clk)
    # whole-job rate: one graph (and the config's R right-hand sides) per job — strong
    # scaling over row partitions (R = 1) or over the split right-hand sides (R > 1)
    value = nnz * R_cfg * M / (ms_step * 1e-3) / 1e9

    # dominant kernel: the fused term kernel (+ its hub-row finalize), from the same
    # graph-replayed solve the step runs (difference of M-term and 0-term replays)
    term_us, tM, t0ms = sv.term_us_replayed(flush, max(3, args.steps // 2))
    term_us = dist.max(term_us)
    vbytes = 8 if args.precision == 64 else 4
    rp_bytes = 8 if info["row_ptr_64"] else 4
    B = algorithmic_bytes(n, nnz, rp_bytes, vbytes, R)
    peak, peak_kind = peaks()
    achieved = B / (term_us * 1e-6) / 1e9
    win = window_info(dg) if R == 1 and dist.world == 1 else None

    exchange_info = None
    if dist.world > 1 and R_cfg == 1:
        # exchange volume per rank per term: the halo push stores x_{k+1}[u] only on the ranks
        # that own a neighbour of u; NCCL all-gathers every slot
        from paper_2112_01743_b200.distributed import partition_info
        pi = partition_info(dg)
        vb = 8 if args.precision == 64 else 4
        if px is not None:
            sent = dist.max(float(pi["halo_stores"] * vb))
        else:
            sent = float((dist.world - 1) * pi["max_rows"] * vb)
        exchange_info = {"scheme": "fused push, halo-only" if px is not None else "NCCL all-gather",
                         "partition": "block-cyclic (snake order) over the degree-sorted rows",
                         "bytes_per_rank_per_term_max": int(sent),
                         "replicate_all_bytes_per_rank": int(pi["all_stores"] * vb),
                         "rows_max": int(dist.max(float(pi["rows"]))), "nnz_local_max": int(dist.max(float(pi["nnz_local"]))),
                         "nvlink_peak_gbs": 770.0,
                         "nvlink_frac_of_term": round(sent / (term_us * 1e-6) / 770e9, 4)}

    comparator = None
    if dist.world == 1 and R == 1 and not args.no_e2e:
        comparator = power_comparator(dg, flush, args.precision)
    e2e = None if args.no_e2e else sv.e2e(device, args.steps, flush, dist, exchange, args.warmup)
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(sv, args.config, args)
    secondary = []
    if dist.world == 1 and args.secondary:
        own = f"{args.config}:{args.precision}"
        for name in [s for s in args.secondary.split(",") if s and s != args.config and s != own]:
            try:
                secondary.append(secondary_line(name, device, args.precision, args.steps, args.warmup, dist))
            except Exception as ex:  # noqa: BLE001
                secondary.append({"config": name, "failed": f"{type(ex).__name__}: {ex}"})

    if dist.rank == 0:
        kernel = ("k_spmm_term + k_spmm_hub_finalize" if R > 1 else
                  ("k_window_pass + " if win else "") + "k_term_warp<EPI_CPAA> + k_hub_finalize")
        clk_summary = clk.summary()
        line = {
            "metric": "cpaa_gteps_per_term",
            "value": round(value, 3),
            "unit": "GTEPS",
            "n_gpus": dist.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "strong" if dist.world > 1 else "weak",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == 64 else "f32",
            "data": "synthetic",
            "config": config_dict(args.config, n, nnz, M, R_cfg),
            "parallelism": (f"rowpart{dist.world}+" + ("push" if px is not None else "nccl_allgather"))
                           if dist.world > 1 and R_cfg == 1 else (f"replicas{dist.world}" if dist.world > 1 else "single"),
            "details": {"edges_drawn": info["edges_drawn"], "max_degree": info["max_degree"],
                        "time_to_1e-10_ms": round(ms_step, 4), "graph_build_s": round(build_s, 3),
                        "gteps_definition": "nnz*R*terms/step_time (every CSR entry one traversal)",
                        "R_per_rank": R,
                        **({"column_windows": win} if win else {}),
                        **({"exchange_note": exchange_note} if exchange_note else {})},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": measured_traffic(args.config, args.precision, dist.world),
                         "traffic_unit": "DRAM bytes per term, summed over the term's kernels "
                                         "(ncu --set full, profiles/traffic.json)",
                         "kernel": kernel, "bytes_per_launch": B,
                         "bytes_formula": "4 nnz + I_r (n+1) + 6 V R n (SURVEY.md 8d)",
                         "mean_launch_us": round(term_us, 3),
                         "launch_timing": f"(t_replay(M={M}) {tM:.4f} ms - t_replay(M=0) {t0ms:.4f} ms) / M, "
                                          "graph-replayed PDL chain, L2 flushed, CUDA events",
                         "peak_kind": peak_kind},
            "cpu_baseline": cpu,
            "e2e": e2e,
            **({"power_comparator": comparator} if comparator else {}),
            **({"exchange": exchange_info} if exchange_info else {}),
            **({"secondary": secondary} if secondary else {}),
            "gpu_launches": launches,
            "clocks": clk_summary,
            "lsu_roofline": lsu_roofline(args.config, args.precision, dist.world, term_us,
                                         clk_summary.get("sm_mhz")),
        }
        print(json.dumps(line))
    dg.free()
    if px is not None:
        px.detach()
    if comm is not None:
        comm.close()
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Benchmark of the CPAA hot path (BASELINE.json metric: GTEPS per Chebyshev term and
time-to-1e-10 on B200, with the HBM-roofline fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--precision 64]
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

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------------------
# clocks sampling during the timed region
# ----------------------------------------------------------------------------------------
class Clocks:
    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

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
        for ln in self.lines:
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
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------
# inputs
# ----------------------------------------------------------------------------------------
def make_edges(cfg: dict, device):
    from paper_2112_01743_b200 import generate as G
    if cfg["kind"] == "gnp":
        e = G.gnp_edges(cfg["n"], cfg["p"], cfg["seed"])
        return e.astype(np.int32) if device is not None else e
    if cfg["kind"] == "chung_lu":
        return G.chung_lu_edges(cfg["n"], cfg["gamma"], cfg["wmin"], cfg["wmax"], cfg["draws"],
                                cfg["seed"], device=device)
    return G.rmat_edges(cfg["scale"], cfg["ef"], 0.57, 0.19, 0.19, cfg["seed"], device=device)


def build_device(cfg: dict, device: int):
    """Generate on the device and run the K1 builder there (no host round trip)."""
    import paper_2112_01743_b200 as cheb
    from paper_2112_01743_b200 import _lib as L
    lib = L.load()
    e = make_edges(cfg, device)
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
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------------------
# reference arm / cpu baseline (the reference compiled unmodified: oracle/_ref)
# ----------------------------------------------------------------------------------------
def cpu_reference_run(cfg: dict, steps: int, warmup: int, threads: int, host_edges=None):
    from oracle import Reference
    ref = Reference()
    e = host_edges if host_edges is not None else make_edges(cfg, None)
    e64 = np.ascontiguousarray(np.asarray(e, dtype=np.int64).reshape(-1, 2))
    t0 = time.perf_counter()
    rg = ref.build_graph(e64, dedup=True, drop_isolated=cfg.get("drop", False))
    build_s = time.perf_counter() - t0
    M, _ = ref.plan_iterations(DAMPING, EPS)
    walls = []
    for i in range(warmup + steps):
        r = rg.run_cpaa(c=DAMPING, eps=EPS, parallelism=threads)
        if i >= warmup:
            walls.append(r.wall_ms)
    return dict(n=rg.n, nnz=rg.nnz, M=M, wall_ms=walls, build_s=build_s)


def run_reference_arm(args):
    cfgname = args.config
    cfg = CONFIGS[cfgname]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    try:
        from oracle import REF_SO
        if not os.path.exists(REF_SO):
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return 0
        threads = os.cpu_count() or 1
        res = cpu_reference_run(cfg, args.steps, args.warmup, threads)
    except Exception as ex:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"{type(ex).__name__}: {ex}"}))
        return 0
    ms = statistics.mean(res["wall_ms"])
    gteps = res["nnz"] * res["M"] / (ms * 1e-3) / 1e9
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
        "config": {"workload": cfgname, "desc": cfg["desc"], "n": res["n"], "nnz": res["nnz"],
                   "terms": res["M"], "eps": EPS, "c": DAMPING, "parallelism": f"cpu{threads}"},
        "cpu_baseline": {"value": round(gteps, 6), "unit": "GTEPS", "cores": threads,
                         "kind": "reference",
                         "sample": f"{cfgname}: one full run_cpaa (M={res['M']}, eps 1e-10) per step, "
                                   f"build excluded ({res['build_s']:.1f}s)"},
        "e2e": {"value": round(gteps, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="build + a few solves, no timing output (for ncu captures)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile_only else args.warmup

    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import paper_2112_01743_b200 as cheb
    from paper_2112_01743_b200 import _lib as L

    dist = Dist(args.gpus)
    device = dist.local
    torch.cuda.set_device(device)
    cfg = CONFIGS[args.config]
    lib = L.load()

    t0 = time.perf_counter()
    dg, info = build_device(cfg, device)
    build_s = time.perf_counter() - t0
    n, nnz = info["n"], info["nnz"]
    M = cheb.plan_iterations(DAMPING, EPS).M
    opts = L.cheb_cpaa_opts()
    lib.cheb_cpaa_opts_default(C.byref(opts))
    opts.eps = EPS
    opts.c = DAMPING
    opts.precision = args.precision
    d_ranks = C.c_void_p()

    def solve():
        cheb.api._check(lib.cheb_cpaa_device(dg.handle, C.byref(opts), C.byref(d_ranks), 0))

    def step_ms():
        lm, tm, terms, launches = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        cheb.api._check(lib.cheb_last_timing(dg.handle, C.byref(lm), C.byref(tm), C.byref(terms),
                                             C.byref(launches)))
        return lm.value, launches.value

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    for _ in range(args.warmup):
        solve()
        step_ms()
    if args.profile_only:
        torch.cuda.synchronize()
        log(f"profile-only: n={n} nnz={nnz} built in {build_s:.2f}s")
        return 0

    dist.barrier()
    torch.cuda.synchronize()
    times, launches = [], 0
    with Clocks(device) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            solve()
            ms, nl = step_ms()
            times.append(ms)
            launches += nl
    torch.cuda.synchronize()
    dist.barrier()
    total_ms = dist.max(sum(times))
    ms_step = total_ms / args.steps
    value = dist.world * nnz * M / (ms_step * 1e-3) / 1e9

    # dominant kernel: the fused term kernel, per-launch CUDA-event durations
    cap = 64
    term_ms = (C.c_double * cap)()
    terms = C.c_int()
    flush.zero_()
    torch.cuda.synchronize()
    cheb.api._check(lib.cheb_cpaa_profile(dg.handle, C.byref(opts), term_ms, cap, C.byref(terms)))
    tms = [term_ms[i] for i in range(terms.value)]
    steady = tms[1:] if len(tms) > 1 else tms
    mean_term = statistics.mean(steady)
    vbytes = 8 if args.precision == 64 else 4
    rp_bytes = 8 if info["row_ptr_64"] else 4
    B = algorithmic_bytes(n, nnz, rp_bytes, vbytes)
    peak, peak_kind = peaks()
    achieved = B / (mean_term * 1e-3) / 1e9

    # e2e through the reference-facing C-ABI with host buffers (pinned), every step
    e2e = None
    if not args.no_e2e:
        host = dg.download()
        off = torch.from_numpy(host.offsets).pin_memory().numpy()
        nb = torch.from_numpy(host.neighbors).pin_memory().numpy()
        deg = host.degrees
        inv = host.inv_degree
        ranks = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
        tr = (L.cheb_trace_row * 64)()
        rounds, tot = C.c_int(), C.c_double()

        def e2e_step():
            h = C.c_void_p()
            cheb.api._check(lib.cheb_graph_upload_csr(
                off.ctypes.data_as(L.I64P), off.size, nb.ctypes.data_as(L.I64P), nb.size,
                deg.ctypes.data_as(L.I64P), deg.size, inv.ctypes.data_as(L.F64P), inv.size,
                n, int(host.m), 0, device, int(info["row_ptr_64"]), C.byref(h)))
            cheb.api._check(lib.cheb_cpaa(h, C.byref(opts), None, 0, ranks.ctypes.data_as(L.F64P),
                                          tr, C.byref(rounds), C.byref(tot)))
            lib.cheb_graph_free(h)

        e2e_step()
        dist.barrier()
        e2e_times = []
        for _ in range(max(1, min(args.steps, 5))):
            flush.zero_()
            torch.cuda.synchronize()
            t = time.perf_counter()
            e2e_step()
            e2e_times.append(time.perf_counter() - t)
        e2e_s = dist.max(statistics.mean(e2e_times))
        e2e = {"value": round(dist.world * nnz * M / e2e_s / 1e9, 4), "unit": "GTEPS",
               "h2d_bytes_per_step": int(off.nbytes + nb.nbytes),
               "d2h_bytes_per_step": int(ranks.nbytes + 2 * M * 8),
               "ms_per_step": round(e2e_s * 1e3, 3),
               "path": "cheb_graph_upload_csr(pinned int64 CSR) + cheb_cpaa(host ranks) + free"}

    # CPU baseline: the reference compiled unmodified, same graph, all host threads
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        try:
            host = dg.download()
            e = np.stack([np.repeat(np.arange(host.n), np.diff(host.offsets)), host.neighbors], 1)
            e = e[e[:, 0] <= e[:, 1]]
            threads = os.cpu_count() or 1
            r = cpu_reference_run(dict(cfg, drop=False), 1, 0, threads, host_edges=e)
            cms = statistics.mean(r["wall_ms"])
            cpu = {"value": round(r["nnz"] * r["M"] / (cms * 1e-3) / 1e9, 6), "unit": "GTEPS",
                   "cores": threads, "kind": "reference",
                   "sample": f"one full run_cpaa (M={r['M']}) on the same {args.config} CSR "
                             f"({r['nnz']} entries), K={threads} threads, wall {cms:.0f} ms"}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "GTEPS", "cores": 0, "kind": "reference",
                   "sample": f"failed: {type(ex).__name__}: {ex}"}

    if dist.rank == 0:
        line = {
            "metric": "cpaa_gteps_per_term",
            "value": round(value, 3),
            "unit": "GTEPS",
            "n_gpus": dist.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == 64 else "f32",
            "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "n": n, "nnz": nnz,
                       "edges_drawn": info["edges_drawn"], "max_degree": info["max_degree"],
                       "terms": M, "eps": EPS, "c": DAMPING,
                       "time_to_1e-10_ms": round(ms_step, 4),
                       "parallelism": "replicas" if dist.world > 1 else "single",
                       "l2": "flushed (512 MiB write) before every timed step",
                       "graph_build_s": round(build_s, 3)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "k_term_fast<EPI_CPAA>", "bytes_per_launch": B,
                         "mean_launch_us": round(mean_term * 1e3, 3), "peak_kind": peak_kind},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    dg.free()
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())

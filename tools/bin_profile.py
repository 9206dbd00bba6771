"""Per-degree-bin evidence for the term kernel (north star: warp efficiency per degree bin,
L2 hit rate on the x-gather).  Run under ncu once per bin with CHEB_TUNE_SKIP=16+b (the term
kernel then processes only tile bin b; b = 0..5 pack tiles with 2^b lanes per row, 6 chunk
tiles of rows above the warp tile), then summarise:
    python tools/bin_profile.py run   [config]   # on the GPU box: ncu captures -> gpurun_out/bins/
    python tools/bin_profile.py table [config]   # here: table from the captures + bin sizes
Skipped tiles still stream their column ids and row operands (the prefetch runs ahead of
the filter), so per-bin DRAM bytes are not attributable; time, warp efficiency and the
hit rates of the LSU gathers are.
The nogather / skip / skipwarm / prefetch / streamcs knobs act only in the experiment build
(`touch paper_2112_01743_b200/csrc/term.cuh && make EXP=1`); the product build compiles them out."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out", "bins")
METRICS = ["gpu__time_duration.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
           "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def bins(cfg):
    sys.path.insert(0, ROOT)
    import ctypes as C
    import numpy as np
    import bench
    from paper_2112_01743_b200 import _lib as L
    dg, info = bench.build_device(bench.CONFIGS[cfg], 0)
    t, r, z = (np.zeros(7, dtype=np.int64) for _ in range(3))
    rc = L.load().cheb_graph_view_bins(dg.handle, t.ctypes.data_as(L.I64P), r.ctypes.data_as(L.I64P),
                                       z.ctypes.data_as(L.I64P))
    assert rc == 0
    return t.tolist(), r.tolist(), z.tolist()


def run(cfg):
    os.makedirs(OUT, exist_ok=True)
    t, r, z = bins(cfg)
    json.dump({"tiles": t, "rows": r, "nnz": z}, open(os.path.join(OUT, f"{cfg}_bins.json"), "w"))
    for b in range(-1, 7):
        env = dict(os.environ)
        if b >= 0:
            env["CHEB_TUNE_SKIP"] = str(16 + b)
        tag = "all" if b < 0 else f"bin{b}"
        cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:k_term_warp",
               "--launch-skip", "20", "-c", "1", "--csv", "--log-file", os.path.join(OUT, f"{cfg}_{tag}.csv"),
               sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "1", "--warmup", "3",
               "--no-cpu-baseline", "--no-e2e"]
        subprocess.run(cmd, env=env, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, check=False)


def table(cfg):
    b = json.load(open(os.path.join(OUT, f"{cfg}_bins.json")))
    print(f"# term kernel per tile bin, {cfg} (tools/bin_profile.py; ncu --clock-control none, one warm launch)")
    print("bin,lanes_per_row,tiles,rows,csr_entries,time_us,G_gathers_per_s,warp_eff_threads_per_inst,"
          "l1_hit_pct,l2_hit_pct_of_l1_misses,lsu_wavefront_pct,warps_active_pct")
    for i in range(-1, 7):
        tag = "all" if i < 0 else f"bin{i}"
        path = os.path.join(OUT, f"{cfg}_{tag}.csv")
        if not os.path.exists(path):
            continue
        rows = [r for r in csv.reader(io.StringIO(open(path).read())) if len(r) > 10]
        hdr = rows[0]
        m = {r[hdr.index("Metric Name")]: r[hdr.index("Metric Value")] for r in rows[1:]}
        val = lambda k: float(m[k].replace(",", ""))  # noqa: E731
        us = val("gpu__time_duration.sum") / 1e3 if "gpu__time_duration.sum" in m else float("nan")
        nnz = sum(b["nnz"]) if i < 0 else b["nnz"][i]
        hit = val("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum") / max(1.0, val("lts__t_sectors_srcunit_tex_op_read.sum"))
        lanes = "mixed" if i < 0 else ("chunk" if i == 6 else str(1 << i))
        tiles = sum(b["tiles"]) if i < 0 else b["tiles"][i]
        rws = sum(b["rows"]) if i < 0 else b["rows"][i]
        print(f"{tag},{lanes},{tiles},{rws},{nnz},{us:.1f},{nnz / (us * 1e-6) / 1e9:.1f},"
              f"{val('smsp__thread_inst_executed_per_inst_executed.ratio'):.2f},"
              f"{val('l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct'):.1f},{100 * hit:.1f},"
              f"{val('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'):.1f},"
              f"{val('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "table"
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
    (run if what == "run" else table)(cfg)

"""Summarise an ncu --set full report (.ncu-rep) into the key roofline/stall figures
committed under profiles/.  Usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1_wavefront_pct"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_read_sectors_from_sm"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1_global_ld_sectors"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_bank_conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "avg_active_threads_per_warp_inst"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1_wavefronts_shared"),
    ("memory_l1_wavefronts_shared_ideal", "l1_wavefronts_shared_ideal"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "l1_wavefronts_global_ld"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1_requests_global_ld"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kre:
        args += ["-k", f"regex:{kre}"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"kernel: {d.get('Kernel Name', '?')}")
        for key, label in KEYS:
            if key in d:
                u = units[hdr.index(key)]
                print(f"  {label:34s} {d[key]} {u}")
        stalls = {k: float(v or 0) for k, v in d.items()
                  if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k)}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda x: -x[1])[:6]
        print("  stall reasons (pc sampling): " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot * 100:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()

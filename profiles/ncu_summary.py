#!/usr/bin/env python
"""Summarise an ncu report (details + raw pages) into the numbers we track.

    python profiles/ncu_summary.py gpurun_out/prof_<tag>.ncu-rep [--raw]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread",
    "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Issued Instructions",
    "Executed Ipc Active", "No Eligible", "Warp Cycles Per Issued Instruction",
    "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput",
    "DRAM Throughput", "Compute (SM) Throughput", "Memory Throughput",
]
RAW = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
    "smsp__pcsamp_warps_issue_stalled_no_instructions",
    "smsp__pcsamp_warps_issue_stalled_branch_resolving",
    "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum",
]


def ncu(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu(rep, "details")
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Unit"), hdr.index("Metric Value"))
    seen = {}
    kernel = None
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        kernel = r[ki]
        if r[mi] in KEYS and r[mi] not in seen:
            seen[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    print(f"kernel: {kernel}")
    for k in KEYS:
        if k in seen:
            print(f"  {k:38s} {seen[k]}")
    raw = ncu(rep, "raw")
    h, u, v = raw[0], raw[1], raw[2]
    d = {a: (b, c) for a, b, c in zip(h, u, v)}
    for k in RAW:
        if k in d:
            print(f"  {k:62s} {d[k][1]} {d[k][0]}")


if __name__ == "__main__":
    main()

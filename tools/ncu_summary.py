#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py full gpurun_out/r01_c2_full.ncu-rep > profiles/r01_c2_force.txt
    python tools/ncu_summary.py launches gpurun_out/r01_launches.csv > profiles/r01_launches.txt

`full`: speed-of-light / occupancy / pipe utilisation / DRAM traffic / stall reasons and the
source lines with the most warp-stall samples (needs -lineinfo builds).
`launches`: per-kernel count, total and mean device time and share of the listed launches.
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

NCU = "/usr/local/cuda/bin/ncu"

KEEP_DETAILS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
                "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
                "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
                "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers",
                "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
                "Branch Efficiency", "Grid Size", "Block Size", "SM Frequency"]
RAW = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
       "smsp__inst_executed.sum", "launch__registers_per_thread",
       "dram__bytes.sum.per_second",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def _csv(args):
    out = subprocess.run([NCU, *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep):
    rows = _csv(["-i", rep, "--page", "details", "--csv"])
    h = rows[0]
    kname, kid = None, None
    print(f"# ncu --set full summary of {rep}")
    for r in rows[1:]:
        rid = r[h.index("ID")] if "ID" in h else None
        if kname is None or rid != kid:
            kname, kid = r[h.index("Kernel Name")], rid
            print(f"kernel [{rid}]: {kname}")
        if r[h.index("Metric Name")] in KEEP_DETAILS:
            print(f"  {r[h.index('Metric Name')]:<40} {r[h.index('Metric Value')]:>14} {r[h.index('Metric Unit')]}")
    raw = _csv(["-i", rep, "--page", "raw", "--csv"])
    h, units, v = raw[0], raw[1], raw[2]
    print("raw:")
    for n in RAW:
        if n in h:
            i = h.index(n)
            print(f"  {n:<70} {v[i]:>16} {units[i]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("stall reasons (warps per issue-active cycle):")
    for x, n in sorted(st, reverse=True)[:10]:
        print(f"  {n:<28} {x:6.2f}")
    src = _csv(["-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"])
    hdr, data = None, []
    for r in src:
        if r and r[0] == "Line No":
            hdr = r
            i_s = hdr.index("Warp Stall Sampling (All Samples)")
            i_ie = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) < len(hdr) or r[2] != "-":
            continue
        try:
            data.append((int(r[i_s]), int(r[i_ie]), int(r[0]), r[1].strip()[:96]))
        except ValueError:
            pass
    if data:
        ts = sum(d[0] for d in data) or 1
        ti = sum(d[1] for d in data) or 1
        print("top source lines (% of stall samples, % of warp instructions):")
        for d in sorted(data, reverse=True)[:25]:
            print(f"  {100 * d[0] / ts:5.1f}% {100 * d[1] / ti:5.1f}%  L{d[2]:<4} {d[3]}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = r[h.index("Kernel Name")]
        agg[k][0] += 1
        agg[k][1] += float(r[h.index("Metric Value")].replace(",", ""))
    tot = sum(t for _, t in agg.values()) or 1
    print(f"# ncu --metrics gpu__time_duration.sum launch list: {path}")
    print(f"# {'launches':>8} {'total_us':>12} {'mean_us':>10} {'share':>7}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {n:>8} {t / 1e3:12.1f} {t / n / 1e3:10.2f} {100 * t / tot:6.1f}%  {k}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])

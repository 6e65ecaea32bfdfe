#!/usr/bin/env python
"""Executed-instruction breakdown of a force-kernel ncu capture by code region (source
line ranges of force_kernel.cuh / ieee_fast.cuh) and opcode.
    python tools/ncu_regions.py gpurun_out/v22/c3_full.ncu-rep"""
import collections
import csv
import io
import re
import subprocess
import sys

REGIONS = [  # (first line of region, name) in force_kernel.cuh, ascending
    (0, "header/helpers"), (170, "jacobi_rot/rot2"), (234, "amax/live/compact"),
    (299, "lmin3_pair sched"), (371, "det_inv"), (422, "pointwise"), (528, "forward_point (stage 3)"),
    (603, "tables/config"), (660, "gather"), (720, "stages 1-2"), (880, "misc modes"),
    (955, "S3 call / dt"), (1030, "S4 backward + S5"), (1300, "assembly")]


def main(rep):
    out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    src = open("paper_2104_11404_b200/csrc/force_kernel.cuh").read().splitlines()
    marks = []
    for i, l in enumerate(src, 1):
        for key, name in (("void jacobi_rot(", "jacobi_rot/rot2"), ("double amax6(", "amax/live/compact"),
                          ("void lmin3_pair(", "lmin3_pair sched"), ("double det_inv(", "det_inv"),
                          ("void pointwise(", "pointwise"), ("void forward_point(", "forward_point (stage 3)"),
                          ("struct Tab24", "tables/config"), ("--- S1 gather", "gather"),
                          ("--- S2 forward", "stages 1-2"), ("--- MODE_FTW", "misc modes"),
                          ("--- S3 pointwise", "S3 call / dt"), ("--- S4 backward", "S4 backward + S5"),
                          ("-- assembly", "assembly")):
            if key in l:
                marks.append((i, name))
    marks.sort()

    def region(f, line):
        if f != "force_kernel.cuh":
            return "ieee_fast (div/sqrt)" if f == "ieee_fast.cuh" else f
        name = "header/helpers"
        for i, n in marks:
            if line is not None and line >= i:
                name = n
        return name
    f = line = None
    agg = collections.defaultdict(collections.Counter)
    tot = 0.0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] in ("Line No", "Function Name"):
            continue
        if r[0] != "":
            line = int(r[0]) if r[0].isdigit() else None
            continue
        m = re.match(r"^\s*(@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_]+)", r[3])
        try:
            ex = float(r[7])
        except ValueError:
            continue
        if not m:
            continue
        agg[region(f, line)][m.group(2)] += ex
        tot += ex
    print(f"# {rep}: {tot:.4g} warp instructions executed")
    for reg, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        s = sum(c.values())
        if s == 0:
            continue
        fp = c["DFMA"] + c["DMUL"] + c["DADD"]
        top = ", ".join(f"{k}:{v / s * 100:.0f}%" for k, v in c.most_common(5))
        print(f"{reg:26s} {s / tot * 100:5.1f}%  fp64 {fp / s * 100:4.0f}%   {top}")
    # whole kernel: opcode totals (warp instructions), FP64-pipe opcodes first
    allc = collections.Counter()
    for c in agg.values():
        allc.update(c)
    d_ops = {k: v for k, v in allc.items() if k.startswith("D") and k not in ("DEPBAR",)}
    print("FP64-pipe opcodes (warp instructions): " +
          ", ".join(f"{k} {v:.4g}" for k, v in sorted(d_ops.items(), key=lambda kv: -kv[1])))
    print("top opcodes: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in allc.most_common(14)))


if __name__ == "__main__":
    main(sys.argv[1])

#!/usr/bin/env python
"""Shared-memory wavefronts per source line of an ncu capture (excessive = bank conflicts):
    python tools/ncu_smem.py REP.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, top=25):
    out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    f = None
    line = None
    agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0] != "":
            line = r[0]
            src = r[1]
            agg[(f, line)][3] = src[:90]
            continue
        d = dict(zip(hdr, r))
        try:
            w = float(d["L1 Wavefronts Shared"]); x = float(d["L1 Wavefronts Shared Excessive"])
            i = float(d["L1 Wavefronts Shared Ideal"])
        except (KeyError, ValueError):
            continue
        a = agg[(f, line)]
        a[0] += w; a[1] += x; a[2] += i
    tot = sum(v[0] for v in agg.values()); ex = sum(v[1] for v in agg.values())
    print(f"# {rep}: shared wavefronts {tot:.4g}, excessive {ex:.4g}")
    for (fn, ln), (w, x, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        if w == 0:
            continue
        print(f"{fn}:{ln:<5} wf {w:10.4g} excess {x:10.4g} ideal {i:10.4g}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

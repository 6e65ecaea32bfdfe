#!/usr/bin/env python
"""Executed warp instructions per source line of one file in an ncu capture (with opcode mix).
    python tools/ncu_lines.py REP.ncu-rep force2d_pl.cuh [top]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, fname, top=40):
    out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    f = line = None
    agg = collections.defaultdict(collections.Counter)
    files = collections.Counter()
    tot = 0.0
    for r in csv.reader(io.StringIO(out)):
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
        tot += ex
        files[f] += ex
        if f == fname:
            agg[line][m.group(2)] += ex
    print(f"# {rep}: {tot:.4g} warp instructions; by file: " +
          ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in files.most_common()))
    for ln, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(c.values())
        print(f"L{ln:<5} {s / tot * 100:5.1f}%  " + ", ".join(f"{k}:{v:.3g}" for k, v in c.most_common(6)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)

#!/usr/bin/env python
"""Record the force kernel's DRAM traffic per launch from ncu --set full captures into
profiles/traffic.json (read by bench.py for the roofline's "traffic" field).

    python tools/traffic.py c1=gpurun_out/v8/c1_full.ncu-rep c2=gpurun_out/v9/c2_full.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "traffic.json")


def read(rep):
    out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def get(name):
        i = h.index(name)
        return float(v[i].replace(",", "")) * scale[units[i]]
    return {"dram_read": get("dram__bytes_read.sum"), "dram_write": get("dram__bytes_write.sum"),
            "kernel": v[h.index("Kernel Name")]}


def main():
    d = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for arg in sys.argv[1:]:
        name, rep = arg.split("=", 1)
        r = read(rep)
        d[name] = {"bytes_per_launch": r["dram_read"] + r["dram_write"], "dram_read": r["dram_read"],
                   "dram_write": r["dram_write"], "kernel": r["kernel"],
                   "source": f"ncu --set full, {os.path.basename(os.path.dirname(rep))}/{os.path.basename(rep)}"}
    json.dump(d, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""A/B timing of several builds of libhydro.so on the same box: each (library, config)
pair runs in its own process (tools/ab.py's timing loop, default kernel selection), the
library order rotating every round.

    python tools/ab_lib.py ROUNDS c1,c2 LIB_A LIB_B [LIB_C ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rounds, cfgs, libs = int(sys.argv[1]), sys.argv[2].split(","), sys.argv[3:]
    for r in range(rounds):
        order = libs[r % len(libs):] + libs[:r % len(libs)]
        for c in cfgs:
            for lib in order:
                env = dict(os.environ, HYDRO_LIB_PATH=os.path.abspath(lib))
                out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab.py"), c,
                                      "HYDRO_AB=1"], env=env, capture_output=True, text=True)
                line = (out.stdout.strip().splitlines() or [out.stderr.strip()[-300:]])[-1]
                print(f"round {r} {os.path.basename(lib)}: {line}", flush=True)


if __name__ == "__main__":
    main()

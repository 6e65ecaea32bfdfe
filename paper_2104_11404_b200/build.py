"""Build libhydro.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2104_11404_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false.
-fmad=false is part of the evaluation contract (DESIGN A.0): the dt-relevant
arithmetic must not be contracted into FMAs behind the source's back; every FMA the
kernels want is written as __fma_rn.  tables.cpp is host code compiled by g++ (it
uses IEEE binary128 for the 1D tables).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libhydro.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["hydro_api.cu"]
SOURCES_CPP = ["tables.cpp"]
HEADERS = ["force_kernel.cuh", "force2d.cuh", "force2d_pl.cuh", "fom.cuh", "ieee_fast.cuh", "rom_kernels.cuh", "offline.cuh", "hydro_internal.h"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "hydro.h")]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
                   "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            with open(os.path.join(BUILD, src + ".ptxas.log"), "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            subprocess.check_call(["g++", "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off",
                                   "-c", s, "-o", o])
    if force or _newer(LIB, objs):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs,
                               "-Xlinker", "--no-undefined"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

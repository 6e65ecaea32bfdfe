#!/usr/bin/env python
"""A/B timing of the C4 GEMM-shaped calls at full size on random data (no C4 problem build):
hydro_rom_project for the velocity (n 40, s 409 866) and energy (n 40, s 41 944) rows and
hydro_rom_lift for the x (3.54 M rows) and e (0.86 M rows, per-instance offsets) fields;
CUDA events, L2 flushed, median of 20.  HYDRO_LIB_PATH selects the library build.
    python tools/gemm_bench.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2104_11404_b200 import hydro
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    r = lambda *sh: torch.randn(*sh, generator=g, device=dev, dtype=torch.float64)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    B, n = 64, 40

    def timed(fn, k=20):
        fn()
        ts = []
        for _ in range(k):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts)) * 1e3
    out = []
    for name, s in (("project_v", 410031), ("project_e", 41944)):
        P, f = r(n, s), r(s, B)
        ws = hydro.rom_project_workspace(n, s, B, dev)
        o = torch.empty((n, B), dtype=torch.float64, device=dev)
        us = timed(lambda: hydro.rom_project(P, f, out=o, workspace=ws))
        err = float((o - P @ f).abs().max() / (P.abs() @ f.abs()).max())
        out.append(f"{name}: {us:.1f} us (rel err {err:.1e})")
    # the same product with the operator stored transposed (Phi^T X, hydro_basis_tproduct; synchronous)
    PT, f = r(410031, n), r(410031, B)
    us = timed(lambda: hydro.basis_tproduct(PT, f))
    out.append(f"tproduct_v: {us:.1f} us")
    for name, rows, batched in (("lift_x", 3544689, False), ("lift_e", 859904, True)):
        Phi, Y = r(rows, n), r(n, B)
        os_ = r(rows, B) if batched else r(rows)
        o = torch.empty((rows, B), dtype=torch.float64, device=dev)
        us = timed(lambda: hydro.rom_lift(Phi, os_, Y, out=o))
        out.append(f"{name}: {us:.1f} us")
    print("  ".join(out))


if __name__ == "__main__":
    main()

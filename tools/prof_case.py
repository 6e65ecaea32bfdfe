#!/usr/bin/env python
"""Short driver for ncu captures: one workload, `--iters` calls of the hot path.

    python tools/prof_case.py c2 --iters 3

Launch order per call (full mode): force_kernel, assemble_kernel.  The context's
m_q setup launch (force_kernel<...,MODE_MQ>) comes first, so `ncu -k regex:force_kernel
-s 2` skips the setup launch and the first (cold) call.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["c0", "c1", "c2", "c3", "c4", "tg"])
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--k2d", default="auto", help="2D Q2 kernel (hydro_set_2d_kernel)")
    a = ap.parse_args()
    import workloads as W
    from paper_2104_11404_b200 import hydro
    hydro.set_kernel_2d(a.k2d)

    dev = torch.device("cuda", 0)
    t = lambda arr, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(arr)).to(dev, dt).contiguous()
    if a.workload == "c4":
        b = W.c4()
        base = b.base
    else:
        base = W.config(a.workload)
    m = base.mesh
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, t(m.elem_nodes, torch.int32), t(m.x0), t(m.rho0))
    visc = hydro.Visc(base.q1, base.q2, base.visc)
    cfl = hydro.Cfl(base.alpha, base.alpha_mu)
    gamma = t(base.gamma)
    if a.workload != "c4":
        x, v, e = t(base.x), t(base.v), t(base.e)
        for _ in range(a.iters):
            F1, FTw, dt = ctx.force_full(x, v, e, gamma, visc, cfl)
    else:
        plan = hydro.SamplePlan(ctx, b.sample_elems, b.B)
        Phi_x, Phi_v, Phi_e = t(b.Phi_x), t(b.Phi_v), t(b.Phi_e)
        x_os, v_os, e_os = t(b.x_os), t(b.v_os), t(b.e_os)
        Yx, Yv, Ye = t(b.Yx), t(b.Yv), t(b.Ye)
        Pv, Pe, Cxv, cx = hydro.offline_projectors(Phi_x, Phi_v, Phi_e, v_os, *W.sampled_row_maps(b))
        wsv = hydro.rom_project_workspace(b.nv, plan.s_v, b.B, dev)
        wse = hydro.rom_project_workspace(b.ne, plan.s_e, b.B, dev)
        # the bench's C4 step: 3 lifts, the sampled force, 2 projections, the r_x lift
        for _ in range(a.iters):
            xS = hydro.rom_lift(Phi_x, x_os, Yx)
            vS = hydro.rom_lift(Phi_v, v_os, Yv)
            eS = hydro.rom_lift(Phi_e, e_os, Ye)
            F1r, FTr, dt = plan.force_sampled(xS, vS, eS, gamma, visc, cfl)
            hydro.rom_project(Pv, F1r, workspace=wsv)
            hydro.rom_project(Pe, FTr, workspace=wse)
            hydro.rom_lift(Cxv, cx, Yv)
    torch.cuda.synchronize()
    st = ctx.status_sync() if a.workload != "c4" else plan.status_sync()
    assert st[0] == 0, st
    print(f"{a.workload}: ok ({a.iters} calls)")


if __name__ == "__main__":
    main()

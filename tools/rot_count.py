#!/usr/bin/env python
"""Jacobi rotation slots executed per warp vs rotations the lanes needed, on a config
(diagnostic library built with -DHYDRO_COUNT_ROT: bash tools/build_variant.sh rotcount
-DHYDRO_COUNT_ROT; run with HYDRO_LIB_PATH=paper_2104_11404_b200/_build/var/rotcount.so).
    python tools/rot_count.py c2"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import workloads as W
    from paper_2104_11404_b200 import hydro
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
    prob = W.c4() if name == "c4" else W.config(name)
    base = prob.base if name == "c4" else prob
    m = base.mesh
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, t(m.elem_nodes, torch.int32), t(m.x0), t(m.rho0))
    g = t(base.gamma)
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
    if name == "c4":
        plan = hydro.SamplePlan(ctx, prob.sample_elems, prob.B)
        xS = hydro.rom_lift(t(prob.Phi_x), t(prob.x_os), t(prob.Yx))
        vS = hydro.rom_lift(t(prob.Phi_v), t(prob.v_os), t(prob.Yv))
        eS = hydro.rom_lift(t(prob.Phi_e), t(prob.e_os), t(prob.Ye))
        run = lambda: plan.force_sampled(xS, vS, eS, g, visc, cfl)
        nqp = plan.n_cl * prob.B * m.nq ** m.dim
    else:
        x, v, e = t(prob.x), t(prob.v), t(prob.e)
        run = lambda: ctx.force_full(x, v, e, g, visc, cfl)
        nqp = m.n_elem * m.nq ** m.dim
    L = hydro.lib()
    f = L.hydro_debug_rot_counts
    f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    c = (ctypes.c_ulonglong * 12)()
    f(c, 1)
    run()
    torch.cuda.synchronize()
    f(c, 1)
    print(f"{name}: lane-slots executed {c[0]}  needed {c[1]}  per point: executed "
          f"{c[0] / nqp:.3f} needed {c[1] / nqp:.3f}  (2 eigen-solves per point)  "
          f"utilisation {c[1] / max(c[0], 1):.3f}")
    print(f"  IEEE re-runs: {c[10]} points ({c[10] / nqp:.2e} of all), in {c[11]} warps")
    for sw in range(4):
        live, ex = c[2 + 2 * sw], c[3 + 2 * sw]
        print(f"  sweep {sw + 1}: matrices live per point {live / nqp:.3f} (of 2), "
              f"lane-slots executed per point {ex / nqp:.3f}")


if __name__ == "__main__":
    main()

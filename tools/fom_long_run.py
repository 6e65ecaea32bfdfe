#!/usr/bin/env python
"""A long full-order run on the GPU as physical evidence at full size: the Taylor-Green
state (workloads "tg", 64^3 Q2/Q1, 6.4 M kinematic dofs) advanced with hydro_fom_advance
under the paper's controller for a fixed simulated time; reports steps,
rejections, wall time per step and the drift of the discrete total energy
1/2 v^T M_V v + 1^T M_E e, which the RK2-average scheme conserves exactly up to
the CG tolerance.  CFL alpha = 0.25 = 0.5/k: with the literal h = sigma_min(J) of DESIGN R2
(not divided by the order, unlike Laghos) the paper's alpha = 0.5 lets the controller run
Q2 at the edge of stability, and both the oracle and this library blow up within ~10 steps
(DESIGN R27).     python tools/fom_long_run.py [t_final_in_initial_dt_units] [alpha]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import workloads as W
    from paper_2104_11404_b200 import hydro
    units = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
    alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
    dev = torch.device("cuda", 0)
    prob = W.config("tg")
    m = prob.mesh
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
    bc = []
    for c in range(m.dim):
        on = np.isclose(m.x0[c], m.lo[c]) | np.isclose(m.x0[c], m.hi[c])
        bc.append(c * m.n_nodes + np.nonzero(on)[0])
    bc = np.sort(np.concatenate(bc)).astype(np.int64)
    v0 = prob.v.copy()
    v0.reshape(-1)[bc] = 0.0
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, t(m.elem_nodes, torch.int32), t(m.x0), t(m.rho0))
    fom = hydro.Fom(ctx, bc)
    x, v, e, g = t(prob.x), t(v0), t(prob.e), t(prob.gamma)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(alpha, prob.alpha_mu)
    dt0 = float(ctx.dt_estimate(x, v, e, g, visc, cfl).item())
    E0 = sum(fom.energy(v, e))
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    tr, h, ns, nr = 0.0, 0.5 * dt0, 0, 0
    trace = []
    while tr < units * dt0:
        t1, h, a, r = fom.advance(x, v, e, g, visc, cfl, tr, units * dt0, h, max_steps=10)
        ns, nr, tr = ns + a, nr + r, t1
        trace.append((tr, h, a, r, sum(fom.energy(v, e))))
        if a == 0:
            break
    torch.cuda.synchronize()
    print(json.dumps({"trace": [[float(a) for a in r] for r in trace]}), file=sys.stderr)
    wall = time.perf_counter() - w0
    E1 = sum(fom.energy(v, e))
    print(json.dumps({"workload": "tg 64^3 Q2/Q1 FOM", "cfl_alpha": alpha, "t_final": tr, "initial_dt_estimate": dt0,
                      "accepted_steps": ns, "rejected_steps": nr, "wall_s": wall,
                      "ms_per_accepted_step": wall / max(ns, 1) * 1e3,
                      "rel_total_energy_drift": abs(E1 - E0) / abs(E0),
                      "status": ctx.status_sync()[0]}))


if __name__ == "__main__":
    main()

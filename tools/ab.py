#!/usr/bin/env python
"""A/B timing of kernel variants, one process, CUDA events, L2 flushed between calls.
A variant K2D=<auto|element|point|lane> selects the 2D Q2 kernel (hydro_set_2d_kernel); any
other NAME=VALUE is set in the environment.

    python tools/ab.py c1 K2D=element K2D=lane
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import workloads as W
    from paper_2104_11404_b200 import hydro
    name, variants = sys.argv[1], sys.argv[2:]
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
    prob = W.c4() if name == "c4" else W.config(name)
    base = prob.base if name == "c4" else prob
    m = base.mesh
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, t(m.elem_nodes, torch.int32), t(m.x0), t(m.rho0))
    g = t(base.gamma)
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
    if name == "c4":
        # the sampled force call of C4 (lifted state fixed); returns (F1 rows, FTw rows, dt)
        plan = hydro.SamplePlan(ctx, prob.sample_elems, prob.B)
        xS = hydro.rom_lift(t(prob.Phi_x), t(prob.x_os), t(prob.Yx))
        vS = hydro.rom_lift(t(prob.Phi_v), t(prob.v_os), t(prob.Yv))
        eS = hydro.rom_lift(t(prob.Phi_e), t(prob.e_os), t(prob.Ye))

        class _C:
            def force_full(self, *a):
                return plan.force_sampled(xS, vS, eS, g, visc, cfl)

            def status_sync(self):
                return plan.status_sync()
        ctx = _C()
        x = v = e = None
    else:
        x, v, e = t(prob.x), t(prob.v), t(prob.e)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    ref = None
    for var in variants:
        k, val = var.split("=")
        if k == "K2D":
            hydro.set_kernel_2d(val)
        else:
            os.environ[k] = val
        for _ in range(3):
            F1, FTw, dt = ctx.force_full(x, v, e, g, visc, cfl)
        torch.cuda.synchronize()
        ts = []
        for _ in range(int(os.environ.get("AB_ITERS", "40"))):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            F1, FTw, dt = ctx.force_full(x, v, e, g, visc, cfl)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        st = ctx.status_sync()
        out = (F1.cpu().numpy(), FTw.cpu().numpy(), float(dt.reshape(-1)[0].item()))
        same = None if ref is None else (np.array_equal(out[1], ref[1]) and out[2] == ref[2])
        ref = ref or out
        print(f"{name} {var}: median {np.median(ts) * 1e3:.1f} us  min {min(ts) * 1e3:.1f}  status {st[0]}  "
              f"dt {out[2]!r}  FTw/dt identical to first variant: {same}")


if __name__ == "__main__":
    main()

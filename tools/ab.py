#!/usr/bin/env python
"""A/B timing of kernel variants selected by env vars (HYDRO_2D_KERNEL, HYDRO_3D_KERNEL),
one process, CUDA events, L2 flushed between calls.

    python tools/ab.py c3 HYDRO_3D_KERNEL=element HYDRO_3D_KERNEL=persistent
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
    prob = W.config(name)
    m = prob.mesh
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, t(m.elem_nodes, torch.int32), t(m.x0), t(m.rho0))
    x, v, e, g = t(prob.x), t(prob.v), t(prob.e), t(prob.gamma)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    ref = None
    for var in variants:
        k, val = var.split("=")
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
        out = (F1.cpu().numpy(), FTw.cpu().numpy(), float(dt.item()))
        same = None if ref is None else (np.array_equal(out[1], ref[1]) and out[2] == ref[2])
        ref = ref or out
        print(f"{name} {var}: median {np.median(ts) * 1e3:.1f} us  min {min(ts) * 1e3:.1f}  status {st[0]}  "
              f"dt {out[2]!r}  FTw/dt identical to first variant: {same}")


if __name__ == "__main__":
    main()

"""Shared glue for the -m gpu tests: move a workloads.Problem to the device, call the
C ABI through the binding, and compare with the oracle under DESIGN "Tolerances"."""
from __future__ import annotations

import numpy as np
import torch

import workloads as W
from paper_2104_11404_b200 import hydro

TOL_ASSEMBLED = 1e-11   # BASELINE north_star: assembled FP64 vectors
TOL_LOCAL = 1e-12       # element-local vectors and sampled rows


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype).contiguous()


def context(prob: W.Problem) -> hydro.HydroContext:
    m = prob.mesh
    return hydro.HydroContext(m.dim, m.k, m.nq, dev(m.elem_nodes, torch.int32), dev(m.x0), dev(m.rho0))


def run_full(prob: W.Problem, ctx=None, w=None):
    ctx = ctx or context(prob)
    F1, FTw, dt = ctx.force_full(dev(prob.x), dev(prob.v), dev(prob.e), dev(prob.gamma),
                                 hydro.Visc(prob.q1, prob.q2, prob.visc),
                                 hydro.Cfl(prob.alpha, prob.alpha_mu),
                                 w=None if w is None else dev(w))
    torch.cuda.synchronize()
    st = ctx.status_sync()
    return dict(F1=F1.cpu().numpy(), FTw=FTw.cpu().numpy(), dt=float(dt.cpu().item()),
                status=st[0], first_bad=st[1], ctx=ctx)


def assert_close(got, ref, mag, tol, what=""):
    got, ref, mag = np.asarray(got), np.asarray(ref), np.asarray(mag)
    scale = np.maximum(np.abs(ref), mag)
    err = np.abs(got - ref)
    bad = err > tol * scale
    if bad.any():
        i = np.argmax(err / np.maximum(scale, 1e-300))
        raise AssertionError(f"{what}: {bad.sum()} entries exceed tol {tol}; worst rel "
                             f"{(err / np.maximum(scale, 1e-300)).ravel()[i]:.3e} "
                             f"got {got.ravel()[i]!r} ref {ref.ravel()[i]!r}")
    return float((err / np.maximum(scale, 1e-300)).max()) if err.size else 0.0


def dt_bitwise(a: float, b: float) -> bool:
    return np.float64(a).tobytes() == np.float64(b).tobytes()


def gpu_offline_ops(batch):
    """The offline operators of a ROM batch formed by the library on the GPU
    (hydro.offline_projectors: hydro_gappy_pinv + hydro_window_ops) -- device tensors
    (P_v, P_e, C_xv, c_x).  The oracle side uses oracle.rom.offline_projectors."""
    h1, l2 = W.sampled_row_maps(batch)
    return hydro.offline_projectors(dev(batch.Phi_x), dev(batch.Phi_v), dev(batch.Phi_e),
                                    dev(batch.v_os), h1, l2)

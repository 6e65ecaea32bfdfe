"""The two-pass F^T w (hydro_force_full_store + hydro_force_transpose and their sampled
forms) against the one-pass hydro_force_full with the same w and against the oracle:
FTw within the element-local tolerance (1e-12 of max(|ref|, M)), F.1 and dt of the store
call identical to hydro_force_full's (same kernel, bitwise)."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from tests import gpu_helpers as H  # noqa: E402
from paper_2104_11404_b200 import hydro  # noqa: E402


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
@pytest.mark.parametrize("kern2d", ["element", "point"])
def test_store_then_transpose(oracle_lib, set_kernel_2d, name, kern2d):
    set_kernel_2d(kern2d)
    prob = W.small(name)
    rng = np.random.default_rng(11)
    w = np.ascontiguousarray(prob.v + 0.05 * rng.standard_normal(prob.v.shape))
    ctx = H.context(prob)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    x, v, e, g = H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma)
    F1s, _, dts, S = ctx.force_full_store(x, v, e, g, visc, cfl)
    F1, _, dt = ctx.force_full(x, v, e, g, visc, cfl)
    assert torch.equal(F1s, F1) and torch.equal(dts, dt)
    FTw = ctx.force_transpose(S, H.dev(w)).cpu().numpy()
    prob.w = w
    ref = oracle_lib.force(prob)
    H.assert_close(FTw, ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, f"{name} transpose FTw")


def test_sampled_store_then_transpose(oracle_lib):
    from tests.test_gpu_rom import oracle_instance
    batch = W.c4(n_sample=6, B=3, small_mesh=True)
    base = batch.base
    ctx = H.context(base)
    plan = hydro.SamplePlan(ctx, batch.sample_elems, batch.B)
    L = hydro.lib()
    xS = hydro.rom_lift(H.dev(batch.Phi_x), H.dev(batch.x_os), H.dev(batch.Yx))
    vS = hydro.rom_lift(H.dev(batch.Phi_v), H.dev(batch.v_os), H.dev(batch.Yv))
    eS = hydro.rom_lift(H.dev(batch.Phi_e), H.dev(batch.e_os), H.dev(batch.Ye))
    wS = (vS * 1.1).contiguous()
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
    F1 = torch.empty((plan.s_v, batch.B), dtype=torch.float64, device="cuda")
    FT = torch.empty((plan.s_e, batch.B), dtype=torch.float64, device="cuda")
    FT2 = torch.empty_like(FT)
    dt = torch.empty(batch.B, dtype=torch.float64, device="cuda")
    S = torch.empty(L.hydro_sample_stress_bytes(plan._h) // 8, dtype=torch.float64, device="cuda")
    import ctypes
    assert L.hydro_force_sampled_store(plan._h, hydro._ptr(xS), hydro._ptr(vS), hydro._ptr(eS),
                                       hydro._ptr(H.dev(base.gamma)), visc.c(), cfl.c(), hydro._ptr(F1),
                                       hydro._ptr(FT), hydro._ptr(dt), hydro._ptr(S),
                                       hydro._stream(None)) == 0
    assert L.hydro_sample_force_transpose(plan._h, hydro._ptr(S), hydro._ptr(wS), hydro._ptr(FT2),
                                          hydro._stream(None)) == 0
    torch.cuda.synchronize()
    FT2 = FT2.cpu().numpy()
    # oracle: F^T w rows with w = 1.1 v
    for b in range(batch.B):
        m = base.mesh
        d, ncl, ne = m.dim, batch.closure_nodes.size, m.ne
        x = m.x0.copy(); x[:, batch.closure_nodes] = xS.cpu().numpy()[:, b].reshape(d, ncl)
        v = np.zeros_like(m.x0); v[:, batch.closure_nodes] = vS.cpu().numpy()[:, b].reshape(d, ncl)
        e = base.e.copy(); e[batch.closure_elems] = eS.cpu().numpy()[:, b].reshape(-1, ne)
        r = oracle_lib.force(base, elist=batch.closure_elems, x=x, v=v, e=e, w=1.1 * v)
        ref = r["FTw"][batch.sample_elems].reshape(-1)
        mag = r["FTwmag"][batch.sample_elems].reshape(-1)
        H.assert_close(FT2[:, b], ref, mag, H.TOL_LOCAL, f"sampled transpose b={b}")

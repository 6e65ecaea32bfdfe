"""GPU parity of the hyper-reduced ROM RK2-average online step (SURVEY 8(f) NEXT-2,
PAPER Eq. RK2-avg-rom-hr) against oracle/rom.py on a C4-shaped batch (3D Q2
sample mesh, B instances with their own energy offsets and per-instance dt): reduced
coordinates after two steps within 1e-10 (relative to their scale), stage dt estimates
within 1e-10 (the lifted states differ at the rounding level of the two GEMM orders, so
dt is not compared bitwise here; the sampled force itself is bit-exact in dt given equal
inputs, tests/test_gpu_rom.py).  The offline operators use the M-orthonormal-basis option
of P:716-723 (Mhat = I): R_v = (Z^T Phi_v)^+, R_e = (Z^T Phi_e)^+."""
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
from oracle import rom as orom  # noqa: E402


@pytest.mark.parametrize("dim", [3, 2])
def test_rom_step_matches_oracle(dim):
    if dim == 3:
        batch = W.c4(n_sample=6, B=3, small_mesh=True)
    else:
        batch = W.rom_batch(W.small("c0"), B=3, n_sample=5, n_red=8)
    base = batch.base
    P_v, P_e, C_xv, c_x = orom.offline_projectors(batch)
    ctx = H.context(base)
    plan = hydro.SamplePlan(ctx, batch.sample_elems, batch.B)
    st = hydro.RomStepper(plan, H.dev(batch.Phi_x), H.dev(batch.Phi_v), H.dev(batch.Phi_e),
                          H.dev(batch.x_os), H.dev(batch.v_os), H.dev(batch.e_os),
                          *H.gpu_offline_ops(batch))
    op = dict(base=base, closure_elems=batch.closure_elems, closure_nodes=batch.closure_nodes,
              s0_nodes=batch.s0_nodes, sample_elems=batch.sample_elems, Phi_x=batch.Phi_x,
              Phi_v=batch.Phi_v, Phi_e=batch.Phi_e, x_os=batch.x_os, v_os=batch.v_os,
              e_os=batch.e_os, R_v=P_v, R_e=P_e, C_xv=C_xv, c_x=c_x)
    Yx, Yv, Ye = H.dev(batch.Yx), H.dev(batch.Yv), H.dev(batch.Ye)
    rx, rv, re = batch.Yx.copy(), batch.Yv.copy(), batch.Ye.copy()
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
    g = H.dev(base.gamma)
    # per-instance steps: a fraction of each instance's own stability estimate
    _, _, _, dt0 = orom.rom_rk2avg_step(op, rx, rv, re, np.zeros(batch.B))
    dt = 0.2 * dt0 * (1.0 + 0.1 * np.arange(batch.B))
    for _ in range(2):
        dte = st.step(Yx, Yv, Ye, g, visc, cfl, H.dev(dt))
        rx, rv, re, dte_ref = orom.rom_rk2avg_step(op, rx, rv, re, dt)
        assert plan.status_sync()[0] == 0
        np.testing.assert_allclose(dte.cpu().numpy(), dte_ref, rtol=1e-10)
    for got, want, what in ((Yx, rx, "xhat"), (Yv, rv, "vhat"), (Ye, re, "ehat")):
        g_ = got.cpu().numpy()
        assert np.abs(g_ - want).max() <= 1e-10 * np.abs(want).max(), what
    # the state moved
    assert np.abs(rv - batch.Yv).max() > 0


def test_rom_step_instances_independent():
    """Instance b of a batch steps exactly like a B = 1 plan of that instance."""
    batch = W.c4(n_sample=4, B=3, small_mesh=True)
    base = batch.base
    P_v, P_e, C_xv, c_x = H.gpu_offline_ops(batch)
    ctx = H.context(base)
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
    g = H.dev(base.gamma)
    dt = np.full(batch.B, 2e-5)

    def run(B, sl):
        plan = hydro.SamplePlan(ctx, batch.sample_elems, B)
        st = hydro.RomStepper(plan, H.dev(batch.Phi_x), H.dev(batch.Phi_v), H.dev(batch.Phi_e),
                              H.dev(batch.x_os), H.dev(batch.v_os),
                              H.dev(np.ascontiguousarray(batch.e_os[:, sl])), P_v, P_e, C_xv, c_x)
        Y = [H.dev(np.ascontiguousarray(a[:, sl])) for a in (batch.Yx, batch.Yv, batch.Ye)]
        st.step(*Y, g, visc, cfl, H.dev(np.ascontiguousarray(dt[sl])))
        torch.cuda.synchronize()
        return [y.cpu().numpy() for y in Y]

    full = run(batch.B, slice(0, batch.B))
    one = run(1, slice(1, 2))
    for a, b in zip(full, one):
        assert np.array_equal(a[:, 1], b[:, 0])


def test_rom_advance_controller_matches_oracle():
    """hydro_rom_advance (P:549-566 controller per instance) against oracle/rom.advance on a
    C4-shaped batch whose instances start from 3x / 0.5x / 1.5x their stability estimates:
    the same per-instance accepted/rejected counts and times, reduced coordinates within
    1e-10 of their scale."""
    batch = W.c4(n_sample=6, B=3, small_mesh=True)
    base = batch.base
    P_v, P_e, C_xv, c_x = orom.offline_projectors(batch)
    ctx = H.context(base)
    plan = hydro.SamplePlan(ctx, batch.sample_elems, batch.B)
    st = hydro.RomStepper(plan, H.dev(batch.Phi_x), H.dev(batch.Phi_v), H.dev(batch.Phi_e),
                          H.dev(batch.x_os), H.dev(batch.v_os), H.dev(batch.e_os),
                          *H.gpu_offline_ops(batch))
    op = dict(base=base, closure_elems=batch.closure_elems, closure_nodes=batch.closure_nodes,
              s0_nodes=batch.s0_nodes, sample_elems=batch.sample_elems, Phi_x=batch.Phi_x,
              Phi_v=batch.Phi_v, Phi_e=batch.Phi_e, x_os=batch.x_os, v_os=batch.v_os,
              e_os=batch.e_os, R_v=P_v, R_e=P_e, C_xv=C_xv, c_x=c_x)
    _, _, _, est0 = orom.rom_rk2avg_step(op, batch.Yx, batch.Yv, batch.Ye, np.zeros(batch.B))
    dt0 = est0 * np.array([3.0, 0.5, 1.5])
    t_final = 2.5 * float(est0.max())
    Yx, Yv, Ye = H.dev(batch.Yx), H.dev(batch.Yv), H.dev(batch.Ye)
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
    tg, hg, nsg, nrg, itg = st.advance(Yx, Yv, Ye, H.dev(base.gamma), visc, cfl, 0.0, t_final,
                                       dt0, max_iters=12)
    rx, rv, re, tr, hr, nsr, nrr, itr = orom.advance(op, batch.Yx.copy(), batch.Yv.copy(),
                                                     batch.Ye.copy(), 0.0, t_final, dt0,
                                                     max_iters=12)
    assert plan.status_sync()[0] == 0
    assert itg == itr and list(nsg) == list(nsr) and list(nrg) == list(nrr)
    assert nrg.sum() > 0 and nsg.sum() > 0
    np.testing.assert_allclose(tg, tr, rtol=1e-12)
    np.testing.assert_allclose(hg, hr, rtol=1e-10)
    for got, want, what in ((Yx, rx, "xhat"), (Yv, rv, "vhat"), (Ye, re, "ehat")):
        g_ = got.cpu().numpy()
        assert np.abs(g_ - want).max() <= 1e-10 * np.abs(want).max(), what


def test_rom_windowed_advance_matches_oracle():
    """Two time windows: window 1 with the batch's bases up to t1, the
    transition Eq. ic-tw into window 2's bases (W.next_window: 24 shared directions), then
    window 2 up to t2 -- against oracle/rom.windowed_advance: per-window step counts, times,
    and the final reduced coordinates within 1e-10 of their scale."""
    b1 = W.c4(n_sample=6, B=3, small_mesh=True)
    b2 = W.next_window(b1)
    base = b1.base
    ctx = H.context(base)
    plan = hydro.SamplePlan(ctx, b1.sample_elems, b1.B)
    g = H.dev(base.gamma)
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)

    def ops(b):
        P_v, P_e, C_xv, c_x = orom.offline_projectors(b)
        op = dict(base=base, closure_elems=b.closure_elems, closure_nodes=b.closure_nodes,
                  s0_nodes=b.s0_nodes, sample_elems=b.sample_elems, Phi_x=b.Phi_x, Phi_v=b.Phi_v,
                  Phi_e=b.Phi_e, x_os=b.x_os, v_os=b.v_os, e_os=b.e_os, R_v=P_v, R_e=P_e,
                  C_xv=C_xv, c_x=c_x)
        st = hydro.RomStepper(plan, H.dev(b.Phi_x), H.dev(b.Phi_v), H.dev(b.Phi_e), H.dev(b.x_os),
                              H.dev(b.v_os), H.dev(b.e_os), *H.gpu_offline_ops(b))
        return op, st
    op1, st1 = ops(b1)
    op2, st2 = ops(b2)
    # the transition operators on the GPU (hydro_window_ops, Eq. ic-tw over the closure rows)
    def trans_ops(f):
        T, c = hydro.window_ops(H.dev(getattr(b2, f"Phi_{f}")), H.dev(getattr(b1, f"Phi_{f}")),
                                H.dev(getattr(b2, f"{f}_os")), H.dev(getattr(b1, f"{f}_os")))
        return T, (c.reshape(-1).contiguous() if getattr(b1, f"{f}_os").ndim == 1 else c)
    dtr = tuple(trans_ops(f) for f in ("x", "v", "e"))
    _, _, _, est0 = orom.rom_rk2avg_step(op1, b1.Yx, b1.Yv, b1.Ye, np.zeros(b1.B))
    dt0 = 0.7 * est0
    t1, t2 = 2.0 * float(est0.max()), 4.0 * float(est0.max())
    ref = orom.windowed_advance([dict(op=op1, t_end=t1), dict(op=op2, t_end=t2)],
                                b1.Yx.copy(), b1.Yv.copy(), b1.Ye.copy(), 0.0, dt0, max_iters=20)
    got = hydro.rom_windowed_advance([dict(stepper=st1, t_end=t1, trans=dtr),
                                      dict(stepper=st2, t_end=t2)],
                                     H.dev(b1.Yx), H.dev(b1.Yv), H.dev(b1.Ye), g, visc, cfl, 0.0,
                                     dt0, max_iters=20)
    assert plan.status_sync()[0] == 0
    for (nsg, nrg), (nsr, nrr) in zip(got[5], ref[5]):
        assert list(nsg) == list(nsr) and list(nrg) == list(nrr)
    np.testing.assert_allclose(got[3], ref[3], rtol=1e-12)
    np.testing.assert_allclose(got[4], ref[4], rtol=1e-10)
    for gt, want, what in zip(got[:3], ref[:3], ("xhat", "vhat", "ehat")):
        g_ = gt.cpu().numpy()
        assert np.abs(g_ - want).max() <= 1e-10 * np.abs(want).max(), what


def test_rom_windowed_advance_previous_offsets_matches_oracle():
    """Time windows with previous-window offsets (Eq. previous_os): window 2's
    offsets are the per-instance lifts of window 1's final state (hydro_rom_window_offset), its
    coordinates restart at 0 and c_x = Phi_x^T v_os per instance (hydro_basis_tproduct) --
    against oracle/rom.windowed_advance(offsets="previous"): per-window step counts and times,
    final coordinates within 1e-10 of their scale; the offsets themselves against the
    oracle's lift of the GPU's window-1 state; the transition's cost recorded."""
    b1 = W.c4(n_sample=6, B=3, small_mesh=True)
    b2 = W.next_window(b1)
    base = b1.base
    ctx = H.context(base)
    plan = hydro.SamplePlan(ctx, b1.sample_elems, b1.B)
    g = H.dev(base.gamma)
    visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)

    def op_of(b):
        P_v, P_e, C_xv, c_x = orom.offline_projectors(b)
        return dict(base=base, closure_elems=b.closure_elems, closure_nodes=b.closure_nodes,
                    s0_nodes=b.s0_nodes, sample_elems=b.sample_elems, Phi_x=b.Phi_x, Phi_v=b.Phi_v,
                    Phi_e=b.Phi_e, x_os=b.x_os, v_os=b.v_os, e_os=b.e_os, R_v=P_v, R_e=P_e,
                    C_xv=C_xv, c_x=c_x)

    def win_of(b, t_end):
        P_v, P_e, C_xv, _ = H.gpu_offline_ops(b)
        return dict(Phi_x=H.dev(b.Phi_x), Phi_v=H.dev(b.Phi_v), Phi_e=H.dev(b.Phi_e), R_v=P_v, R_e=P_e,
                    C_xv=C_xv, t_end=t_end)
    op1, op2 = op_of(b1), op_of(b2)
    _, _, _, est0 = orom.rom_rk2avg_step(op1, b1.Yx, b1.Yv, b1.Ye, np.zeros(b1.B))
    dt0 = 0.7 * est0
    t1, t2 = 2.0 * float(est0.max()), 4.0 * float(est0.max())
    ref = orom.windowed_advance([dict(op=op1, t_end=t1), dict(op=op2, t_end=t2)], b1.Yx.copy(),
                                b1.Yv.copy(), b1.Ye.copy(), 0.0, dt0, max_iters=20, offsets="previous")
    cx0 = H.gpu_offline_ops(b1)[3]
    got = hydro.rom_windowed_advance_previous(
        plan, [win_of(b1, t1), win_of(b2, t2)], H.dev(b1.x_os), H.dev(b1.v_os), H.dev(b1.e_os), cx0,
        H.dev(b1.Yx), H.dev(b1.Yv), H.dev(b1.Ye), g, visc, cfl, 0.0, dt0, max_iters=20)
    assert plan.status_sync()[0] == 0
    for (nsg, nrg), (nsr, nrr) in zip(got[5], ref[5]):
        assert list(nsg) == list(nsr) and list(nrg) == list(nrr)
    np.testing.assert_allclose(got[3], ref[3], rtol=1e-12)
    # window 2's coordinates restart at 0 (the oracle's Eq. ic-tw gives rounding noise there),
    # so compare the lifted states of window 2, os_2 + Phi_2 yhat, relative to each field
    Y1 = orom.windowed_advance([dict(op=op1, t_end=t1)], b1.Yx.copy(), b1.Yv.copy(), b1.Ye.copy(),
                               0.0, dt0, max_iters=20)
    for f, gt, want, Yf in zip("xve", got[:3], ref[:3], Y1[:3]):
        os2 = orom.previous_window_offset(op1[f"Phi_{f}"], op1[f"{f}_os"], Yf)
        a = orom.lift(op2[f"Phi_{f}"], os2, gt.cpu().numpy())
        b_ = orom.lift(op2[f"Phi_{f}"], os2, want)
        assert np.abs(a - b_).max() <= 1e-10 * np.abs(b_).max(), f
    assert len(got[6]) == 1 and got[6][0] > 0
    # the transition on its own: offsets = the lift of the final state, coordinates 0
    Y = [H.dev(a) for a in (b1.Yx, b1.Yv, b1.Ye)]
    os_new, Y0, cx = hydro.rom_previous_window(
        (H.dev(b1.Phi_x), H.dev(b1.Phi_v), H.dev(b1.Phi_e)), (H.dev(b1.x_os), H.dev(b1.v_os), H.dev(b1.e_os)),
        Y, (H.dev(b2.Phi_x), H.dev(b2.Phi_v), H.dev(b2.Phi_e)), H.dev(b2.Phi_x))
    for o, P, os_, Yh in zip(os_new, (b1.Phi_x, b1.Phi_v, b1.Phi_e), (b1.x_os, b1.v_os, b1.e_os),
                             (b1.Yx, b1.Yv, b1.Ye)):
        want = orom.previous_window_offset(P, os_, Yh)
        assert np.abs(o.cpu().numpy() - want).max() <= 1e-14 * np.abs(want).max()
    assert all(float(y.abs().max()) == 0.0 for y in Y0)
    cx_want = b2.Phi_x.T @ os_new[1].cpu().numpy()
    assert np.abs(cx.cpu().numpy() - cx_want).max() <= 1e-12 * max(np.abs(cx_want).max(), 1e-30)

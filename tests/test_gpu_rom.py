"""GPU parity of the hyper-reduced ROM online step (C4 shape): lift, sampled force,
projection -- against the oracle's naive lift/projection loops and its element-list
force evaluation per instance (PAPER Sec. 3.3-3.4)."""
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


def oracle_instance(oracle_lib, batch, xS, vS, eS, b):
    base, m = batch.base, batch.base.mesh
    d, ncl, ne = m.dim, batch.closure_nodes.size, m.ne
    x = m.x0.copy()
    x[:, batch.closure_nodes] = xS[:, b].reshape(d, ncl)
    v = np.zeros_like(m.x0)
    v[:, batch.closure_nodes] = vS[:, b].reshape(d, ncl)
    e = base.e.copy()
    e[batch.closure_elems] = eS[:, b].reshape(-1, ne)
    r = oracle_lib.force(base, elist=batch.closure_elems, x=x, v=v, e=e)
    F1 = r["F1"][:, batch.s0_nodes].reshape(-1)
    F1m = r["F1mag"][:, batch.s0_nodes].reshape(-1)
    FT = r["FTw"][batch.sample_elems].reshape(-1)
    FTm = r["FTwmag"][batch.sample_elems].reshape(-1)
    return F1, F1m, FT, FTm, r["dt"]


def gpu_step(batch, ctx=None, plan=None):
    base = batch.base
    ctx = ctx or H.context(base)
    plan = plan or hydro.SamplePlan(ctx, batch.sample_elems, batch.B)
    assert np.array_equal(plan.closure_elems, batch.closure_elems)
    assert np.array_equal(plan.closure_nodes, batch.closure_nodes)
    assert np.array_equal(plan.s0_nodes, batch.s0_nodes)
    xS = hydro.rom_lift(H.dev(batch.Phi_x), H.dev(batch.x_os), H.dev(batch.Yx))
    vS = hydro.rom_lift(H.dev(batch.Phi_v), H.dev(batch.v_os), H.dev(batch.Yv))
    eS = hydro.rom_lift(H.dev(batch.Phi_e), H.dev(batch.e_os), H.dev(batch.Ye))
    F1, FT, dt = plan.force_sampled(xS, vS, eS, H.dev(base.gamma), hydro.Visc(base.q1, base.q2, base.visc),
                                    hydro.Cfl(base.alpha, base.alpha_mu))
    torch.cuda.synchronize()
    st = plan.status_sync()
    return dict(ctx=ctx, plan=plan, xS=xS.cpu().numpy(), vS=vS.cpu().numpy(), eS=eS.cpu().numpy(),
                F1=F1.cpu().numpy(), FT=FT.cpu().numpy(), dt=dt.cpu().numpy(), status=st,
                F1_t=F1, FT_t=FT)


def test_rom_small_lift_force_project(oracle_lib):
    batch = W.c4(n_sample=6, B=5, small_mesh=True)
    g = gpu_step(batch)
    assert g["status"][0] == 0
    # lift vs naive loops
    for key, Phi, os_, Y in (("xS", batch.Phi_x, batch.x_os, batch.Yx), ("vS", batch.Phi_v, batch.v_os, batch.Yv),
                             ("eS", batch.Phi_e, batch.e_os, batch.Ye)):
        ref = oracle_lib.lift(Phi, os_, Y)
        mag = np.abs(os_ if os_.ndim == 2 else os_[:, None]) + np.abs(Phi) @ np.abs(Y)
        H.assert_close(g[key], ref, mag, 1e-14, f"lift {key}")
    # sampled force per instance vs oracle on the closure
    for b in range(batch.B):
        F1, F1m, FT, FTm, dt = oracle_instance(oracle_lib, batch, g["xS"], g["vS"], g["eS"], b)
        H.assert_close(g["F1"][:, b], F1, F1m, H.TOL_LOCAL, f"F1_rows b={b}")
        H.assert_close(g["FT"][:, b], FT, FTm, H.TOL_LOCAL, f"FTw_rows b={b}")
        assert H.dt_bitwise(g["dt"][b], dt)
    # projection (the same oracle-formed operators on both sides: this checks the GEMMs)
    from oracle import rom as orom
    P_v, P_e, C_xv, c_x = orom.offline_projectors(batch)
    rv = hydro.rom_project(H.dev(P_v), g["F1_t"]).cpu().numpy()
    re_ = hydro.rom_project(H.dev(P_e), g["FT_t"]).cpu().numpy()
    H.assert_close(rv, oracle_lib.project(P_v, g["F1"]), np.abs(P_v) @ np.abs(g["F1"]), 1e-13, "r_v")
    H.assert_close(re_, oracle_lib.project(P_e, g["FT"]), np.abs(P_e) @ np.abs(g["FT"]), 1e-13, "r_e")
    rx = hydro.rom_lift(H.dev(C_xv), H.dev(c_x), H.dev(batch.Yv)).cpu().numpy()
    H.assert_close(rx, oracle_lib.lift(C_xv, c_x, batch.Yv), np.abs(C_xv) @ np.abs(batch.Yv), 1e-14, "r_x")


def test_rom_batched_equals_single_and_full():
    """P14: instance b of a batch is bitwise equal to a B=1 plan; sampled rows equal the
    full-order evaluation restricted to S0 (same elements, same ascending order)."""
    batch = W.c4(n_sample=4, B=3, small_mesh=True)
    g = gpu_step(batch)
    base, m = batch.base, batch.base.mesh
    for b in range(batch.B):
        single = W.RomBatch(**{**batch.__dict__, "B": 1, "mu": batch.mu[b:b + 1],
                               "e_os": np.ascontiguousarray(batch.e_os[:, b:b + 1]),
                               "Yx": np.ascontiguousarray(batch.Yx[:, b:b + 1]),
                               "Yv": np.ascontiguousarray(batch.Yv[:, b:b + 1]),
                               "Ye": np.ascontiguousarray(batch.Ye[:, b:b + 1])})
        s = gpu_step(single, ctx=g["ctx"])
        assert np.array_equal(s["xS"][:, 0], g["xS"][:, b])
        assert np.array_equal(s["F1"][:, 0], g["F1"][:, b])
        assert np.array_equal(s["FT"][:, 0], g["FT"][:, b])
        assert s["dt"][0] == g["dt"][b]
        # full-order evaluation on the lifted state
        d, ncl = m.dim, batch.closure_nodes.size
        prob = W.Problem("full", m, m.x0.copy(), np.zeros_like(m.x0), base.e.copy(), base.gamma, True)
        prob.x[:, batch.closure_nodes] = g["xS"][:, b].reshape(d, ncl)
        prob.v[:, batch.closure_nodes] = g["vS"][:, b].reshape(d, ncl)
        prob.e[batch.closure_elems] = g["eS"][:, b].reshape(-1, m.ne)
        full = H.run_full(prob, ctx=g["ctx"])
        assert np.array_equal(full["F1"][:, batch.s0_nodes].reshape(-1), g["F1"][:, b])
        assert np.array_equal(full["FTw"][batch.sample_elems].reshape(-1), g["FT"][:, b])


@pytest.mark.slow
def test_rom_full_size_c4_sampled_instances(oracle_lib):
    """C4 at its BASELINE size (64 instances, 2 % sample of the 64^3 mesh), the bench's launch:
    every instance checked row by row (every sampled F.1 and F^T.v row) against the oracle's
    evaluation over the closure, and its dt bit-exact."""
    batch = W.c4()
    g = gpu_step(batch)
    assert g["status"][0] == 0
    for b in range(batch.B):
        F1, F1m, FT, FTm, dt = oracle_instance(oracle_lib, batch, g["xS"], g["vS"], g["eS"], b)
        H.assert_close(g["F1"][:, b], F1, F1m, H.TOL_LOCAL, f"F1_rows b={b}")
        H.assert_close(g["FT"][:, b], FT, FTm, H.TOL_LOCAL, f"FTw_rows b={b}")
        assert H.dt_bitwise(g["dt"][b], dt)


@pytest.mark.slow
def test_rom_full_size_c4_all_dt_projection_lift(oracle_lib):
    """C4 at its BASELINE size: (a) dt of all 64 instances bit-exact against an oracle dt-only
    pass per instance over the closure (the GPU's lifted state as input); (b) the projection of
    the full sampled rows (s_v = 409 866, s_e = 41 944) against the oracle's naive loops with
    the same offline operators (Eq. sol-ls-hyper); (c) the lift on 20 000 seeded
    closure rows of each field against the oracle's naive lift; (d) the GPU-formed
    offline operators against the oracle's (hydro_gappy_pinv vs numpy pinv)."""
    from oracle import rom as orom
    batch = W.c4()
    g = gpu_step(batch)
    assert g["status"][0] == 0
    base, m = batch.base, batch.base.mesh
    d, ncl, ne = m.dim, batch.closure_nodes.size, m.ne
    for b in range(batch.B):
        x = m.x0.copy()
        x[:, batch.closure_nodes] = g["xS"][:, b].reshape(d, ncl)
        v = np.zeros_like(m.x0)
        v[:, batch.closure_nodes] = g["vS"][:, b].reshape(d, ncl)
        e = base.e.copy()
        e[batch.closure_elems] = g["eS"][:, b].reshape(-1, ne)
        r = oracle_lib.force(base, elist=batch.closure_elems, x=x, v=v, e=e, mode=1)
        assert r["status"] == 0
        assert H.dt_bitwise(g["dt"][b], r["dt"]), (b, g["dt"][b], r["dt"])
    P_v, P_e, C_xv, c_x = orom.offline_projectors(batch)
    rv = hydro.rom_project(H.dev(P_v), g["F1_t"]).cpu().numpy()
    re_ = hydro.rom_project(H.dev(P_e), g["FT_t"]).cpu().numpy()
    H.assert_close(rv, oracle_lib.project(P_v, g["F1"]), np.abs(P_v) @ np.abs(g["F1"]), 1e-13, "r_v full")
    H.assert_close(re_, oracle_lib.project(P_e, g["FT"]), np.abs(P_e) @ np.abs(g["FT"]), 1e-13, "r_e full")
    rng = np.random.default_rng(2104)
    for key, Phi, os_, Y in (("xS", batch.Phi_x, batch.x_os, batch.Yx), ("vS", batch.Phi_v, batch.v_os, batch.Yv),
                             ("eS", batch.Phi_e, batch.e_os, batch.Ye)):
        rows = np.sort(rng.choice(Phi.shape[0], 20_000, replace=False))
        ref = oracle_lib.lift(np.ascontiguousarray(Phi[rows]), np.ascontiguousarray(os_[rows]), Y)
        mag = np.abs(os_[rows] if os_.ndim == 2 else os_[rows][:, None]) + np.abs(Phi[rows]) @ np.abs(Y)
        H.assert_close(g[key][rows], ref, mag, 1e-14, f"lift {key} (full size, sampled rows)")
    got = [t.cpu().numpy() for t in H.gpu_offline_ops(batch)]
    for gg, w, what in zip(got, (P_v, P_e, C_xv, c_x), ("P_v", "P_e", "C_xv", "c_x")):
        assert np.abs(gg - w).max() <= 1e-11 * np.abs(w).max(), what


@pytest.mark.parametrize("n,s,B", [(40, 410031, 64), (40, 409866, 64), (40, 41944, 64), (40, 1000, 64), (40, 997, 64),
                                   (17, 5000, 8), (8, 64, 2), (40, 300, 5), (33, 12345, 7), (64, 3000, 64)])
def test_rom_project_kernel_paths(n, s, B):
    """hydro_rom_project on every kernel path (the cp.async-staged tensor-pipe kernel for even B,
    with 16- or 8-byte copies of P for even / odd s -- C4's s_v = 410 031 is odd --, the
    register-tiled tensor-pipe kernel for odd B, the FP64 FMA fallback for n > 40)
    against the projection's definition r = P f in extended-precision numpy, to
    1e-13 of |P| |f|; and bitwise reproducible."""
    rng = np.random.default_rng(n * 7 + s + B)
    P = rng.standard_normal((n, s))
    f = rng.standard_normal((s, B))
    ref = (P.astype(np.longdouble) @ f.astype(np.longdouble)).astype(np.float64)
    mag = np.abs(P) @ np.abs(f)
    dP, df = H.dev(P), H.dev(f)
    a = hydro.rom_project(dP, df).cpu().numpy()
    b = hydro.rom_project(dP, df).cpu().numpy()
    H.assert_close(a, ref, mag, 1e-13, f"project n={n} s={s} B={B}")
    assert np.array_equal(a, b)

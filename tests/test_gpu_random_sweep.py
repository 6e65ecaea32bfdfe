"""Seeded random sweep of the boundary calls against the oracle: mesh dimension, order,
shape (ragged element counts), node perturbation, velocity pattern, viscosity on/off, w = v
or a separate w, the 2D kernel choice, and -- for the sampled call -- batch size B, sample
size and basis width.  Every case is a pure function of its integer seed (the choices are
drawn from numpy's PCG64 on the test side; the problem data come from workloads/ as
everywhere else), so a failure reproduces with

    python tests/test_gpu_random_sweep.py full SEED      (or: rom SEED, fom SEED, romstep SEED, offline SEED)

and `python tests/test_gpu_random_sweep.py sweep START COUNT [KINDS]` runs a longer sweep of both
kinds (and of two RK2-average FOM steps and two hyper-reduced ROM steps per seed) on the GPU box (seeds START .. START+COUNT-1), printing one line per case.

Bars as everywhere (BASELINE north_star; DESIGN "Tolerances"): F.1 within 1e-11 (assembled)
or 1e-12 (sampled rows), F^T.w within 1e-12 of max(|ref|, M), dt bit-exact."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    if __name__ != "__main__":
        pytest.skip("no CUDA device", allow_module_level=True)

from tests import gpu_helpers as H  # noqa: E402
from paper_2104_11404_b200 import hydro  # noqa: E402


def random_problem(seed: int, rom: bool = False):
    """(problem, description, 2D kernel choice, w or None) of one seed."""
    rng = np.random.default_rng(seed)
    dim = int(rng.integers(2, 4))
    k = int(rng.integers(2, 4))
    nq = 4 if k == 2 else 6
    hi_n = (13 if dim == 2 else 6) if k == 2 else (7 if dim == 2 else 4)
    hi_n *= int(os.environ.get("SWEEP_SCALE", "1"))   # larger meshes for the recorded sweeps
    shape = tuple(int(rng.integers(1, hi_n + 1)) for _ in range(dim))
    kind = "sedov" if rom else ["sedov", "sedov", "gresho", "tg", "triple"][int(rng.integers(0, 5))]
    cfg = 9000 + seed
    if kind == "gresho" and dim == 2:
        prob = W.gresho(cfg, shape, k=k, nq=nq)
    elif kind == "tg" and dim == 3:
        prob = W.taylor_green(cfg, shape, k=k, nq=nq)
    elif kind == "triple" and dim == 3:
        prob = W.triple_point(cfg, shape, hi=tuple(0.25 * s for s in shape), k=k, nq=nq)
    else:
        kind = "sedov"
        h = float(rng.choice([0.01875, 0.125, 1.0]))
        delta = float(rng.choice([0.0, 0.03, 0.1]))
        vmode = str(rng.choice(["uniform", "radial", "zero"]))
        prob = W.sedov_like(cfg, dim, shape, (0.0,) * dim, tuple(h * s for s in shape), delta=delta,
                            e_floor=float(rng.choice([1e-6, 1e-3, 0.5])), vmode=vmode,
                            vscale=float(rng.choice([0.05, 0.5])), k=k, nq=nq, name=f"sweep{seed}")
        kind += f"(h={h},delta={delta},{vmode})"
    if rng.integers(0, 3) == 0:
        prob.visc = not prob.visc
    k2d = str(rng.choice(["auto", "element", "point", "lane"])) if (dim == 2 and k == 2) else "auto"
    w = None
    if not rom and rng.integers(0, 2) == 0:
        w = W.uniform_pm(W.stream_seed(cfg, 77), prob.v.size, 0.3).reshape(prob.v.shape)
    what = f"seed {seed}: {kind} d{dim} Q{k} {shape} visc={prob.visc} k2d={k2d} w={'v' if w is None else 'own'}"
    return prob, what, k2d, w


def run_full_case(oracle_lib, seed: int) -> str:
    prob, what, k2d, w = random_problem(seed)
    hydro.set_kernel_2d(k2d)
    try:
        if w is not None:
            prob.w = w
        ref = oracle_lib.force(prob)
        got = H.run_full(prob, w=w)
    finally:
        hydro.set_kernel_2d("auto")
    assert got["status"] == ref["status"], (what, got["status"], ref["status"])
    if ref["status"] != 0:
        return what + f" -> status {ref['status']} on both sides"
    e1 = H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, f"{what} F1")
    e2 = H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, f"{what} FTw")
    assert H.dt_bitwise(got["dt"], ref["dt"]), (what, got["dt"], ref["dt"])
    return what + f" -> F1 {e1:.1e} FTw {e2:.1e} dt {got['dt']!r}"


def oracle_instance(oracle_lib, batch, xS, vS, eS, b):
    """Instance b of the batch through the oracle: its element-list force evaluation over the
    closure with the lifted state scattered into the full mesh; sampled rows, dt and status."""
    base, m = batch.base, batch.base.mesh
    d, ncl, ne = m.dim, batch.closure_nodes.size, m.ne
    x = m.x0.copy()
    x[:, batch.closure_nodes] = xS[:, b].reshape(d, ncl)
    v = np.zeros_like(m.x0)
    v[:, batch.closure_nodes] = vS[:, b].reshape(d, ncl)
    e = base.e.copy()
    e[batch.closure_elems] = eS[:, b].reshape(-1, ne)
    r = oracle_lib.force(base, elist=batch.closure_elems, x=x, v=v, e=e)
    return dict(F1=r["F1"][:, batch.s0_nodes].reshape(-1), F1m=r["F1mag"][:, batch.s0_nodes].reshape(-1),
                FT=r["FTw"][batch.sample_elems].reshape(-1), FTm=r["FTwmag"][batch.sample_elems].reshape(-1),
                dt=r["dt"], status=r["status"])


def run_rom_case(oracle_lib, seed: int) -> str:
    from tests.test_gpu_rom import gpu_step
    base, what, k2d, _ = random_problem(seed, rom=True)
    rng = np.random.default_rng(100003 + seed)
    m = base.mesh
    E = m.n_elem
    B = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 16, 31, 64]))
    ns = int(rng.integers(1, min(E, 8) + 1))
    # basis width within the smallest possible row counts (ns elements' L2 dofs; one element's nodes)
    n_red = min(int(rng.choice([1, 3, 8, 17, 40])), ns * m.ne, m.dim * (m.k + 1) ** m.dim)
    batch = W.rom_batch(base, cfg=9500 + seed, B=B, n_sample=ns, n_red=n_red)
    what += f" B={B} sample={ns} of {E} n_red={n_red}"
    hydro.set_kernel_2d(k2d)
    try:
        g = gpu_step(batch)
    finally:
        hydro.set_kernel_2d("auto")
    # every instance: dt bit-exact (NaN on both sides when the lifted energy goes negative at a
    # point, DESIGN R12; tangled instances still evaluate, R16); the rows of all finite instances
    worst1 = worst2 = 0.0
    statuses = set()
    for b in range(B):
        o = oracle_instance(oracle_lib, batch, g["xS"], g["vS"], g["eS"], b)
        statuses.add(int(o["status"]))
        if np.isnan(o["dt"]):
            assert np.isnan(g["dt"][b]), (what, b, g["dt"][b])
            continue
        assert H.dt_bitwise(g["dt"][b], o["dt"]), (what, b, g["dt"][b], o["dt"])
        worst1 = max(worst1, H.assert_close(g["F1"][:, b], o["F1"], o["F1m"], H.TOL_LOCAL, f"{what} F1_rows b={b}"))
        worst2 = max(worst2, H.assert_close(g["FT"][:, b], o["FT"], o["FTm"], H.TOL_LOCAL, f"{what} FTw_rows b={b}"))
    # the batch-wide status: 0 iff every instance is clean, else one of the instances' codes
    st = int(g["status"][0])
    assert (st == 0) == (statuses == {0}) and st in statuses, (what, st, statuses)
    # projection of the sampled rows against the plain definition (fp64 numpy product)
    F = np.nan_to_num(g["F1"])
    P = W.uniform_pm(W.stream_seed(9500 + seed, 78), n_red * F.shape[0], 1.0).reshape(n_red, -1)
    r = hydro.rom_project(H.dev(P), H.dev(F)).cpu().numpy()
    H.assert_close(r, P @ F, np.abs(P) @ np.abs(F), 1e-13, f"{what} projection")
    return what + f" -> F1 {worst1:.1e} FTw {worst2:.1e} statuses {sorted(statuses)}"


def run_fom_case(seed: int) -> str:
    """Two RK2-average steps (PAPER Eq. RK2-avg) of a random box problem with a smooth
    positive energy field against oracle/fom.py: states within 1e-11 of their largest entry,
    the step's dt estimate to 1e-10 (tests/test_gpu_fom.py's bars), v.n = 0 rows exactly 0."""
    import oracle
    from oracle import fom as ofom
    rng = np.random.default_rng(200003 + seed)
    dim = int(rng.integers(2, 4))
    k = int(rng.integers(2, 4))
    nq = 4 if k == 2 else 6
    hi_n = (9 if dim == 2 else 4) if k == 2 else (4 if dim == 2 else 2)
    shape = tuple(int(rng.integers(1, hi_n + 1)) for _ in range(dim))
    h = float(rng.choice([0.02, 0.1, 1.0]))
    delta = float(rng.choice([0.0, 0.04, 0.08] if k == 2 else [0.0, 0.02, 0.04]))
    prob = W.sedov_like(9700 + seed, dim, shape, (0.0,) * dim, tuple(h * s for s in shape), delta=delta,
                        e_floor=1e-2, vmode=str(rng.choice(["uniform", "radial"])),
                        vscale=float(rng.choice([0.02, 0.2])) * min(1.0, 10.0 * h), k=k, nq=nq,
                        name=f"fomsweep{seed}")
    prob.e[:] = 1.0 + 0.5 * rng.random(prob.e.shape)
    prob.visc = bool(rng.integers(0, 4) != 0)
    what = f"seed {seed}: fom d{dim} Q{k} {shape} h={h} delta={delta} visc={prob.visc}"
    m = prob.mesh
    bc = ofom.bc_dofs_box(m)
    prob.v.reshape(-1)[bc] = 0.0
    ref = ofom.Fom(m, bc)
    ctx = H.context(prob)
    f = hydro.Fom(ctx, bc)
    x, v, e, g = H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    xr, vr, er = prob.x.copy(), prob.v.copy(), prob.e.copy()
    r0 = oracle.force(prob)
    if r0["status"] != 0:
        return what + f" -> skipped (initial status {r0['status']})"
    dt = float(rng.choice([0.1, 0.25])) * r0["dt"]
    its = 0
    for _ in range(2):
        xr, vr, er, dt_r = ofom.rk2avg_step(ref, prob, xr, vr, er, dt)
        if not np.isfinite(dt_r):
            return what + " -> skipped (the oracle's step leaves the valid states)"
        dt_g, iters = f.step(x, v, e, g, visc, cfl, dt, cg_tol=1e-14, cg_max_iter=4000)
        its += int(np.sum(iters))
        assert ctx.status_sync()[0] == 0, what
        assert abs(dt_g - dt_r) <= 1e-10 * abs(dt_r), (what, dt_g, dt_r)
    worst = 0.0
    for got, want, name in ((x, xr, "x"), (v, vr, "v"), (e, er, "e")):
        err = np.abs(got.cpu().numpy() - want).max() / max(np.abs(want).max(), 1e-300)
        assert err <= 1e-11, (what, name, err)
        worst = max(worst, err)
    assert np.array_equal(v.cpu().numpy().reshape(-1)[bc], np.zeros(bc.size)), what
    return what + f" -> worst {worst:.1e}, {its} CG iterations"


def run_romstep_case(seed: int) -> str:
    """Two hyper-reduced RK2-average ROM steps (PAPER Eq. RK2-avg-rom-hr) of a random
    batch with per-instance dt against oracle/rom.py (tests/test_gpu_rom_step.py's bars: reduced
    coordinates within 1e-10 of their scale, stage dt estimates to 1e-10)."""
    from oracle import rom as orom
    base, what, k2d, _ = random_problem(seed, rom=True)
    rng = np.random.default_rng(300007 + seed)
    m = base.mesh
    E = m.n_elem
    B = int(rng.choice([1, 2, 3, 5, 8]))
    ns = int(rng.integers(1, min(E, 6) + 1))
    # basis width at most half the sampled L2 rows, so the gappy pseudo-inverses stay well conditioned
    n_red = max(1, min(int(rng.choice([1, 2, 4, 8, 12])), (ns * m.ne) // 2))
    batch = W.rom_batch(base, cfg=9800 + seed, B=B, n_sample=ns, n_red=n_red)
    what += f" B={B} sample={ns} of {E} n_red={n_red}"
    P_v, P_e, C_xv, c_x = orom.offline_projectors(batch)
    op = dict(base=base, closure_elems=batch.closure_elems, closure_nodes=batch.closure_nodes,
              s0_nodes=batch.s0_nodes, sample_elems=batch.sample_elems, Phi_x=batch.Phi_x,
              Phi_v=batch.Phi_v, Phi_e=batch.Phi_e, x_os=batch.x_os, v_os=batch.v_os,
              e_os=batch.e_os, R_v=P_v, R_e=P_e, C_xv=C_xv, c_x=c_x)
    rx, rv, re = batch.Yx.copy(), batch.Yv.copy(), batch.Ye.copy()
    _, _, _, dt0 = orom.rom_rk2avg_step(op, rx, rv, re, np.zeros(B))
    if not np.isfinite(dt0).all() or (dt0 <= 0).any():
        return what + " -> skipped (an instance starts tangled or with a negative energy)"
    dt = float(rng.choice([0.1, 0.2])) * dt0 * (1.0 + 0.1 * np.arange(B))
    ctx = H.context(base)
    hydro.set_kernel_2d(k2d)
    try:
        plan = hydro.SamplePlan(ctx, batch.sample_elems, B)
        st = hydro.RomStepper(plan, H.dev(batch.Phi_x), H.dev(batch.Phi_v), H.dev(batch.Phi_e),
                              H.dev(batch.x_os), H.dev(batch.v_os), H.dev(batch.e_os),
                              *H.gpu_offline_ops(batch))
        Yx, Yv, Ye = H.dev(batch.Yx), H.dev(batch.Yv), H.dev(batch.Ye)
        visc, cfl = hydro.Visc(base.q1, base.q2, base.visc), hydro.Cfl(base.alpha, base.alpha_mu)
        g = H.dev(base.gamma)
        for _ in range(2):
            rx, rv, re, dte_ref = orom.rom_rk2avg_step(op, rx, rv, re, dt)
            if not np.isfinite(dte_ref).all():
                return what + " -> skipped (the oracle's step leaves the valid states)"
            dte = st.step(Yx, Yv, Ye, g, visc, cfl, H.dev(dt))
            assert plan.status_sync()[0] == 0, what
            np.testing.assert_allclose(dte.cpu().numpy(), dte_ref, rtol=1e-10, err_msg=what)
    finally:
        hydro.set_kernel_2d("auto")
    worst = 0.0
    for got, want, name in ((Yx, rx, "xhat"), (Yv, rv, "vhat"), (Ye, re, "ehat")):
        err = np.abs(got.cpu().numpy() - want).max() / max(np.abs(want).max(), 1e-300)
        assert err <= 1e-10, (what, name, err)
        worst = max(worst, err)
    return what + f" -> worst {worst:.1e}"


def run_offline_case(seed: int) -> str:
    """The offline selections on a random orthonormal basis: greedy DEIM, Q-DEIM and
    the oversampled greedy must return the oracle's indices exactly; POD of random snapshots with
    a geometric spectrum must return the oracle's basis size, singular values and an orthonormal
    basis (tests/test_gpu_offline.py's bars)."""
    from oracle import offline as ooff
    rng = np.random.default_rng(400009 + seed)
    m = int(rng.choice([1, 2, 3, 7, 16, 33, 40, 64]))
    N = int(rng.integers(m, m + int(rng.choice([4, 300, 30_000]))) + 1)
    n_s = int(rng.integers(m, min(N, 2 * m + 5) + 1))
    U, _ = np.linalg.qr(rng.standard_normal((N, m)))
    U = np.ascontiguousarray(U)
    what = f"seed {seed}: offline N={N} m={m} n_s={n_s}"
    Ud = H.dev(U)
    np.testing.assert_array_equal(hydro.deim(Ud), ooff.deim(U), err_msg=what + " deim")
    np.testing.assert_array_equal(hydro.qdeim(Ud), ooff.qdeim(U), err_msg=what + " qdeim")
    np.testing.assert_array_equal(hydro.deim_oversampled(Ud, n_s), ooff.deim_oversampled(U, n_s),
                                  err_msg=what + " oversampled")
    ns = int(rng.integers(2, 41))
    Np = int(rng.integers(ns, 20_000))
    Q1, _ = np.linalg.qr(rng.standard_normal((Np, ns)))
    Q2, _ = np.linalg.qr(rng.standard_normal((ns, ns)))
    sv = 3.0 / float(rng.choice([1.3, 1.6, 2.5])) ** np.arange(ns)
    S = np.ascontiguousarray(((Q1 * sv) @ Q2.T).T)
    eps = float(rng.choice([0.9, 0.99, 0.9999]))
    Phi_g, sg = hydro.pod(H.dev(S), eps=eps)
    Phi_o, so = ooff.pod(S, eps=eps)
    assert Phi_g.shape == Phi_o.shape, (what, Phi_g.shape, Phi_o.shape)
    tol = 1e-13 * so[0] ** 2 / np.maximum(so, 1e-300) + 1e-12 * so
    assert np.all(np.abs(sg - so) <= tol), (what, float(np.max(np.abs(sg - so) / tol)))
    Pg = Phi_g.cpu().numpy()
    k = Pg.shape[1]
    np.testing.assert_allclose(Pg.T @ Pg, np.eye(k), atol=1e-12, err_msg=what + " pod orthonormality")
    return what + f" pod N={Np} ns={ns} eps={eps} k={k} -> ok"


@pytest.mark.parametrize("seed", range(40))
def test_random_full_force(oracle_lib, seed):
    run_full_case(oracle_lib, seed)


@pytest.mark.parametrize("seed", range(20))
def test_random_sampled_force(oracle_lib, seed):
    run_rom_case(oracle_lib, seed)


@pytest.mark.parametrize("seed", range(12))
def test_random_fom_steps(oracle_lib, seed):
    run_fom_case(seed)


@pytest.mark.parametrize("seed", range(12))
def test_random_rom_steps(oracle_lib, seed):
    run_romstep_case(seed)


@pytest.mark.parametrize("seed", range(10))
def test_random_offline_selections(seed):
    run_offline_case(seed)


if __name__ == "__main__":
    import oracle
    oracle.build()
    mode = sys.argv[1]
    if mode == "full":
        print(run_full_case(oracle, int(sys.argv[2])))
    elif mode == "rom":
        print(run_rom_case(oracle, int(sys.argv[2])))
    elif mode == "fom":
        print(run_fom_case(int(sys.argv[2])))
    elif mode == "romstep":
        print(run_romstep_case(int(sys.argv[2])))
    elif mode == "offline":
        print(run_offline_case(int(sys.argv[2])))
    else:
        start, count = int(sys.argv[2]), int(sys.argv[3])
        kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["full", "rom", "fom", "romstep", "offline"]
        bad = 0
        for s in range(start, start + count):
            for name, fn in (("full", run_full_case), ("rom", run_rom_case),
                             ("fom", lambda o, sd: run_fom_case(sd)),
                             ("romstep", lambda o, sd: run_romstep_case(sd)),
                             ("offline", lambda o, sd: run_offline_case(sd))):
                if name not in kinds:
                    continue
                try:
                    print(name, fn(oracle, s), flush=True)
                except Exception as ex:  # noqa: BLE001
                    bad += 1
                    print(name, f"seed {s} FAILED: {type(ex).__name__}: {str(ex)[:400]}", flush=True)
        print(f"sweep done: {bad} failures")
        sys.exit(1 if bad else 0)

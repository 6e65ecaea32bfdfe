"""Pins of the hyper-reduced ROM-step oracle (oracle/rom.py):

P21 with full bases (Phi = I), a full sample (every element, every row) and the exact
    reduced operators R_v = M_V^{-1}, R_e = M_E^{-1}, C_xv = I, the hyper-reduced
    RK2-average step IS the full-order RK2-average step:
    compared with oracle/fom.py (independent formulation: sparse direct solves, no lift,
    no sampling) over two steps;
P22 lifting with a zero reduced coordinate returns the offset; a unit coordinate returns
    the offset plus that basis column.
"""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W

pytest.importorskip("scipy")


def test_P21_full_basis_rom_step_is_fom_step(oracle_lib):
    from oracle import fom, rom
    prob = W.sedov_like(51, 2, (3, 2), (0.0, 0.0), (0.3, 0.2), delta=0.08, e_floor=1e-2,
                        vmode="uniform", vscale=0.1, name="romfull")
    rng = np.random.default_rng(3)
    prob.e[:] = 1.0 + 0.5 * rng.random(prob.e.shape)
    m = prob.mesh
    F = fom.Fom(m, np.zeros(0, dtype=np.int64))          # no boundary condition
    d, n, E, ne = m.dim, m.n_nodes, m.n_elem, m.ne
    Minv = np.linalg.inv(F.M.toarray())
    R_v = np.kron(np.eye(d), Minv)                       # rows c*n + i (= F1 rows order)
    R_e = np.zeros((E * ne, E * ne))
    for k in range(E):
        R_e[k * ne:(k + 1) * ne, k * ne:(k + 1) * ne] = np.linalg.inv(F.ME[k])
    op = dict(base=prob, closure_elems=np.arange(E, dtype=np.int32),
              closure_nodes=np.arange(n, dtype=np.int64), s0_nodes=np.arange(n, dtype=np.int64),
              sample_elems=np.arange(E, dtype=np.int32),
              Phi_x=np.eye(d * n), Phi_v=np.eye(d * n), Phi_e=np.eye(E * ne),
              x_os=np.zeros(d * n), v_os=np.zeros(d * n), e_os=np.zeros((E * ne, 1)),
              R_v=R_v, R_e=R_e, C_xv=np.eye(d * n), c_x=np.zeros(d * n))
    Yx, Yv, Ye = (prob.x.reshape(-1, 1).copy(), prob.v.reshape(-1, 1).copy(),
                  prob.e.reshape(-1, 1).copy())
    x, v, e = prob.x.copy(), prob.v.copy(), prob.e.copy()
    dt = 0.25 * oracle_lib.force(prob)["dt"]
    for _ in range(2):
        Yx, Yv, Ye, dt_rom = rom.rom_rk2avg_step(op, Yx, Yv, Ye, np.array([dt]))
        x, v, e, dt_fom = fom.rk2avg_step(F, prob, x, v, e, dt)
        assert dt_rom[0] == dt_fom or abs(dt_rom[0] - dt_fom) <= 1e-12 * dt_fom
    assert np.abs(Yx[:, 0] - x.reshape(-1)).max() <= 1e-14 * np.abs(x).max()
    assert np.abs(Yv[:, 0] - v.reshape(-1)).max() <= 1e-12 * np.abs(v).max()
    assert np.abs(Ye[:, 0] - e.reshape(-1)).max() <= 1e-12 * np.abs(e).max()


def test_P22_lift_basis_columns():
    from oracle import rom
    rng = np.random.default_rng(5)
    Phi = rng.standard_normal((30, 4))
    os_ = rng.standard_normal(30)
    Y = np.zeros((4, 3))
    assert np.array_equal(rom.lift(Phi, os_, Y), np.repeat(os_[:, None], 3, axis=1))
    Y[2, 1] = 1.0
    out = rom.lift(Phi, os_, Y)
    assert np.array_equal(out[:, 1], os_ + Phi[:, 2])


def test_P24_rom_controller_is_per_instance():
    """The batched online loop applies the controller of P:549-566 to each instance as if it
    ran alone: with a scripted step whose estimate differs per instance, every instance's
    trial-step sequence, counts and final time equal oracle/fom.advance on that instance
    alone (whose controller trace is pinned by hand in P23); coordinates of a rejected or
    finished instance are left untouched."""
    from oracle import fom, rom
    ests = np.array([1.0, 0.3, 5.0])
    seen = {b: [] for b in range(3)}

    def step(Yx, Yv, Ye, h):
        for b in range(3):
            if h[b] > 0:
                seen[b].append(h[b])
        return Yx + h[None, :], Yv + 2 * h[None, :], Ye - h[None, :], ests.copy()
    Y0 = np.zeros((2, 3))
    Yx, Yv, Ye, t, hn, ns, nr, it = rom.advance(None, Y0, Y0, Y0, 0.0, 3.0, [2.0, 2.0, 2.0],
                                                step=step)
    for b in range(3):
        calls = []

        def one(x, v, e, h):
            calls.append(h)
            return x, v, e, ests[b]
        *_, tb, hb, nsb, nrb = fom.advance(None, None, 0, 0, 0, 0.0, 3.0, 2.0, step=one)
        assert seen[b] == calls
        assert (ns[b], nr[b], t[b], hn[b]) == (nsb, nrb, tb, hb)
        # accepted increments only: x advanced by exactly the accepted steps
        acc = [c for c, nxt in zip(calls, calls[1:] + [None]) if c < ests[b]]
        assert np.isclose(Yx[0, b], sum(acc), rtol=1e-14)
        assert np.isclose(Ye[1, b], -sum(acc), rtol=1e-14)


def test_P25_window_transition():
    """Eq. ic-tw: (a) the same orthonormal basis and offset in both windows ->
    identity; (b) a next-window basis that contains the previous one's span and the same
    offset -> the lifted state is reproduced exactly (up to rounding): os + Phi_w yhat_w =
    os + Phi_{w-1} yhat_{w-1}; (c) different offsets whose difference lies in span(Phi_w) ->
    the lifted state is again reproduced; (d) the factored offline form the GPU path uses,
    T = Phi_w^T Phi_{w-1}, c = Phi_w^T (os_{w-1} - os_w) (oracle.rom.window_transition_ops),
    agrees with the direct formula."""
    from oracle import rom
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((50, 8)))
    Y = rng.standard_normal((8, 3))
    os_ = rng.standard_normal(50)
    np.testing.assert_allclose(rom.window_transition(Q, Q, os_, os_, Y), Y, atol=1e-14)
    Q2, _ = np.linalg.qr(np.concatenate([Q, rng.standard_normal((50, 4))], axis=1))
    Y2 = rom.window_transition(Q2, Q, os_, os_, Y)
    np.testing.assert_allclose(os_[:, None] + Q2 @ Y2, os_[:, None] + Q @ Y, atol=1e-13)
    os2 = os_ + Q2 @ rng.standard_normal(12)
    Y2 = rom.window_transition(Q2, Q, os2, os_, Y)
    np.testing.assert_allclose(os2[:, None] + Q2 @ Y2, os_[:, None] + Q @ Y, atol=1e-12)
    T, c = rom.window_transition_ops(Q2, Q, os2, os_)
    np.testing.assert_allclose(T @ Y + c[:, None], Y2, atol=1e-12)


def _orth(rng, N, k):
    return np.linalg.qr(rng.standard_normal((N, k)))[0]


def test_P35_oblique_transition_with_identity_mass_is_ic_tw():
    """Eq. ic2-tw with M = I and an orthonormal new basis reduces to Eq. ic-tw."""
    from oracle import rom
    rng = np.random.default_rng(35)
    N = 60
    Pn, Po = _orth(rng, N, 5), _orth(rng, N, 4)
    osn, oso = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    Y = rng.standard_normal((4, 3))
    np.testing.assert_allclose(rom.window_transition_oblique(Pn, Po, osn, oso, Y, lambda a: a),
                               rom.window_transition(Pn, Po, osn, oso, Y), atol=1e-13)


def test_P36_oblique_transition_is_an_m_projector():
    """For an SPD M (here a random SPD matrix, and the oracle's own FOM M_V and M_E): a lifted
    state already in os_w + span(Phi_w) maps to its exact coordinates, and in general the
    residual of the new window's lift is M-orthogonal to Phi_w (the Galerkin condition that
    defines an oblique projection) -- a transposed operand or a dropped M fails one of them."""
    from oracle import fom, rom
    rng = np.random.default_rng(36)
    prob = W.sedov_like(36, 2, (3, 2), (0.0, 0.0), (0.3, 0.2), delta=0.08, e_floor=1e-2,
                        vmode="uniform", vscale=0.1, name="obl")
    m = prob.mesh
    Mv = fom.mass_v(m)
    Me = fom.mass_e(m)
    A = rng.standard_normal((40, 40))
    cases = [(40, lambda a: (A @ A.T + 40 * np.eye(40)) @ a),
             (Mv.shape[0], lambda a: Mv @ a),
             (m.n_elem * m.ne, lambda a: np.einsum("eij,ejk->eik", Me,
                                                   a.reshape(m.n_elem, m.ne, -1)).reshape(a.shape))]
    for N, M in cases:
        Pn, Po = _orth(rng, N, 6), _orth(rng, N, 5)
        osn, oso = rng.standard_normal((N, 2)), rng.standard_normal((N, 2))
        z = rng.standard_normal((6, 2))
        # choose Y so that os_old + Phi_old Y - os_new = Phi_new z + (a part outside span(Phi_old))
        Y = rng.standard_normal((5, 2))
        lifted = oso + Po @ Y - osn
        y = rom.window_transition_oblique(Pn, Po, osn, oso, Y, M)
        r = lifted - Pn @ y
        scale = np.abs(Pn.T @ M(lifted)).max()
        np.testing.assert_allclose(Pn.T @ M(r), 0.0, atol=1e-12 * scale)
        # exact reproduction: the old window is the new basis with an offset shifted inside
        # its span, os_old = os_new + Phi_w w, so the lifted state is os_w + Phi_w (w + z)
        w = rng.standard_normal((6, 1))
        y2 = rom.window_transition_oblique(Pn, Pn, osn, osn + Pn @ w, z, M)
        np.testing.assert_allclose(y2, z + w, atol=1e-12 * np.abs(z + w).max())


def test_P37_indicator_vanishes_for_full_bases(oracle_lib):
    """Theorem 2's integrands vanish when the ROM is the FOM: Phi = I, U = I with every row
    sampled (P = I, M Phi Mhat^-1 Phi^T = M M^-1 = I) -- at a real state, through the force
    oracle."""
    from oracle import rom
    prob = W.sedov_like(37, 2, (3, 2), (0.0, 0.0), (0.3, 0.2), delta=0.08, e_floor=1e-2,
                        vmode="uniform", vscale=0.1, name="ind")
    m = prob.mesh
    NV, NE = m.dim * m.n_nodes, m.n_elem * m.ne
    ev, ee = rom.aposteriori_integrand(prob, prob.x, prob.v, prob.e, np.eye(NV), np.eye(NE),
                                       np.eye(NV), np.arange(NV), np.eye(NE), np.arange(NE))
    import oracle
    out = oracle.force(prob, w=prob.v)
    assert ev <= 1e-12 * np.abs(out["F1"]).sum() and ee <= 1e-12 * np.abs(out["FTw"]).sum()


def test_P38_indicator_with_sns_basis_is_the_distance_to_its_span():
    """With the SNS force basis U = M Phi sampled on every row, P is the
    orthogonal projector onto span(M Phi) and M Phi Mhat^-1 Phi^T P = P, so the integrand is
    the Euclidean distance of f from span(M Phi) -- computed independently from an
    orthonormal basis of that span (QR); zero for f inside it."""
    from oracle import rom
    rng = np.random.default_rng(38)
    N, n = 50, 6
    A = rng.standard_normal((N, N))
    Mmat = A @ A.T + N * np.eye(N)
    M = lambda a: Mmat @ a  # noqa: E731
    Phi = np.linalg.qr(rng.standard_normal((N, n)))[0]
    U = Mmat @ Phi
    f = rng.standard_normal(N)
    Q = np.linalg.qr(U)[0]
    dist = np.linalg.norm(f - Q @ (Q.T @ f))
    assert abs(rom.indicator_term(f, Phi, M, U, np.arange(N)) - dist) <= 1e-12 * np.linalg.norm(f)
    g = U @ rng.standard_normal(n)
    assert rom.indicator_term(g, Phi, M, U, np.arange(N)) <= 1e-12 * np.linalg.norm(g)
    # DEIM sampling (n rows) of an SNS basis still reproduces anything in its span exactly
    from oracle import offline
    assert rom.indicator_term(g, Phi, M, U, offline.deim(U)) <= 1e-11 * np.linalg.norm(g)


def test_P42_previous_window_offset_starts_at_zero():
    """Eq. previous_os: with os_w = os_{w-1} + Phi_{w-1} yhat_{w-1}, Eq. ic-tw
    gives yhat_w = 0 (to rounding) for any next-window basis, and the new window's lifted
    state os_w + Phi_w 0 is the previous window's final lift -- "the best approximation of the
    final state in the previous window in the solution subspace of the current window"."""
    from oracle import rom
    rng = np.random.default_rng(42)
    Q1 = _orth(rng, 60, 7)
    Q2 = _orth(rng, 60, 9)                       # unrelated next-window basis
    os1 = rng.standard_normal((60, 4))
    Y1 = rng.standard_normal((7, 4))
    os2 = rom.previous_window_offset(Q1, os1, Y1)
    np.testing.assert_allclose(os2, os1 + Q1 @ Y1, rtol=0, atol=1e-14)
    Y2 = rom.window_transition(Q2, Q1, os2, os1, Y1)
    assert np.abs(Y2).max() <= 1e-14 * np.abs(os2).max()
    np.testing.assert_allclose(rom.lift(Q2, os2, np.zeros((9, 4))), rom.lift(Q1, os1, Y1), atol=1e-14)
    # a shared (1-D) offset becomes per instance
    os2b = rom.previous_window_offset(Q1, os1[:, 0], Y1)
    np.testing.assert_allclose(os2b, os1[:, :1] + Q1 @ Y1, atol=1e-14)


def _small_rom_op(batch):
    from oracle import rom
    P_v, P_e, C_xv, c_x = rom.offline_projectors(batch)
    return dict(base=batch.base, closure_elems=batch.closure_elems, closure_nodes=batch.closure_nodes,
                s0_nodes=batch.s0_nodes, sample_elems=batch.sample_elems, Phi_x=batch.Phi_x,
                Phi_v=batch.Phi_v, Phi_e=batch.Phi_e, x_os=batch.x_os, v_os=batch.v_os,
                e_os=batch.e_os, R_v=P_v, R_e=P_e, C_xv=C_xv, c_x=c_x)


def test_P43_previous_window_offsets_with_equal_bases_continue_the_trajectory(oracle_lib):
    """Two windows with the same bases and previous-window offsets: window 2 restarts from
    yhat = 0 about os_2 = os_1 + Phi yhat(t1), with c_x,2 = Phi_x^T v_os,2 = c_x + C_xv vhat(t1),
    so its reduced dynamics are those of window 1 shifted by a constant and the lifted
    trajectory continues unchanged: the final lifted state equals that of the same bases run
    without a transition (stopped and restarted at t1, the same controller sequence), to
    rounding; step counts agree."""
    from oracle import rom
    batch = W.c4(n_sample=6, B=2, small_mesh=True)
    op = _small_rom_op(batch)
    _, _, _, est0 = rom.rom_rk2avg_step(op, batch.Yx, batch.Yv, batch.Ye, np.zeros(batch.B))
    dt0 = 0.5 * est0
    t1, t2 = 1.5 * float(est0.max()), 3.0 * float(est0.max())
    # reference: one window, stopped and restarted at t1
    Yx, Yv, Ye, _, h, ns1, nr1, _ = rom.advance(op, batch.Yx, batch.Yv, batch.Ye, 0.0, t1, dt0)
    Yx, Yv, Ye, tr, _, ns2, nr2, _ = rom.advance(op, Yx, Yv, Ye, t1, t2, h)
    ref = [rom.lift(op[f"Phi_{f}"], op[f"{f}_os"], Y) for f, Y in zip("xve", (Yx, Yv, Ye))]
    got = rom.windowed_advance([dict(op=op, t_end=t1), dict(op=op, t_end=t2)], batch.Yx, batch.Yv,
                               batch.Ye, 0.0, dt0, offsets="previous")
    # window 2's offsets, as windowed_advance formed them
    Yx1, Yv1, Ye1, *_ = rom.advance(op, batch.Yx, batch.Yv, batch.Ye, 0.0, t1, dt0)
    os2 = [rom.previous_window_offset(op[f"Phi_{f}"], op[f"{f}_os"], Y) for f, Y in zip("xve", (Yx1, Yv1, Ye1))]
    lifted = [rom.lift(op[f"Phi_{f}"], o, Y) for f, o, Y in zip("xve", os2, got[:3])]
    for a, b, what in zip(lifted, ref, ("x", "v", "e")):
        assert np.abs(a - b).max() <= 1e-10 * np.abs(b).max(), what
    np.testing.assert_allclose(got[3], tr, rtol=1e-14)
    assert [list(x) for x in got[5][1]] == [list(ns2), list(nr2)]

"""CPU oracle of the hyper-reduced ROM online step -- TEST INFRASTRUCTURE ONLY
(same import rules as oracle/__init__.py).

PAPER.md Eq. RK2-avg-rom-hr with the lifted approximation
Eq. discretesolrepresentation and the hyper-reduced projection
Eq. sol-ls-hyper:

    vhat^{n+1/2} = vhat^n - (dt/2) R_v f1(U~^n)_S            U~ = (v_os + Phi_v vhat, e_os + Phi_e ehat,
    ehat^{n+1/2} = ehat^n + (dt/2) R_e ftv(U~^n; v~^{n+1/2})_S        x_os + Phi_x xhat)
    xhat^{n+1/2} = xhat^n + (dt/2) (c_x + C_xv vhat^{n+1/2})
    vhat^{n+1}   = vhat^n - dt R_v f1(U~^{n+1/2})_S
    ehat^{n+1}   = ehat^n + dt R_e ftv(U~^{n+1/2}; v~bar)_S,    v~bar = v_os + Phi_v (vhat^n + vhat^{n+1})/2
    xhat^{n+1}   = xhat^n + dt (c_x + C_xv vbarhat)

R_v = Mhat_V^{-1} Phi_v^T Phi_F1 (Z^T Phi_F1)^+ and R_e likewise, C_xv = Phi_x^T Phi_v,
c_x = Phi_x^T v_os are offline operators given to the step; the
subscript S denotes the sampled rows (H1 dofs of the S0 nodes, L2 dofs of the S0
elements; the lifting only on the sample-mesh closure).  Each instance b of a
batch is an independent simulation with its own offsets, coordinates and dt.

The force rows come from oracle.force on the closure elements with the lifted state
written into a full-size state (outside the closure the values are irrelevant: those
elements are not evaluated).  Pinned by tests/test_rom_oracle_pins.py (with full bases
and a full sample, the ROM step is the FOM step of oracle/fom.py).
"""
from __future__ import annotations

import numpy as np

from . import force as _force


def lift(Phi, os_, Y):
    """os + Phi Y, os [rows] or [rows][B]."""
    os2 = os_[:, None] if os_.ndim == 1 else os_
    return os2 + Phi @ Y


def sampled_force(batch_base, closure_elems, closure_nodes, s0_nodes, sample_elems, xS, vS, eS,
                  wS, b):
    """F.1 rows at the S0 nodes and F^T w rows of the S0 elements for instance b."""
    m = batch_base.mesh
    d, ncl, ne = m.dim, closure_nodes.size, m.ne
    x = m.x0.copy()
    x[:, closure_nodes] = xS[:, b].reshape(d, ncl)
    v = np.zeros_like(m.x0)
    v[:, closure_nodes] = vS[:, b].reshape(d, ncl)
    w = np.zeros_like(m.x0)
    w[:, closure_nodes] = wS[:, b].reshape(d, ncl)
    e = batch_base.e.copy()
    e[closure_elems] = eS[:, b].reshape(-1, ne)
    r = _force(batch_base, elist=closure_elems, x=x, v=v, e=e, w=w)
    F1 = r["F1"][:, s0_nodes].reshape(-1)
    FT = r["FTw"][sample_elems].reshape(-1)
    # a tangled or non-finite evaluation makes the instance's estimate NaN (DESIGN R26)
    return F1, FT, (float("nan") if r["status"] else r["dt"])


def offline_projectors(batch):
    """The offline operators of the hyper-reduced step over the sample-mesh rows,
    by their definitions with library primitives (numpy pinv = SVD, matrix products):
    P_v = (Z_v^T Phi_v)^+ [nv][s_v], P_e = (Z_e^T Phi_e)^+ [ne][s_e] (Eq. sol-ls-hyper
    P:778-799, SNS with M = I P:985-1000), C_xv = Phi_x^T Phi_v [nx][nv], c_x = Phi_x^T v_os
    [nx].  The GPU path forms them with hydro_gappy_pinv / hydro_window_ops."""
    import workloads as W
    h1, l2 = W.sampled_row_maps(batch)
    P_v = np.ascontiguousarray(np.linalg.pinv(batch.Phi_v[h1]))
    P_e = np.ascontiguousarray(np.linalg.pinv(batch.Phi_e[l2]))
    C_xv = np.ascontiguousarray(batch.Phi_x.T @ batch.Phi_v)
    c_x = np.ascontiguousarray(batch.Phi_x.T @ batch.v_os)
    return P_v, P_e, C_xv, c_x


def window_transition_ops(Phi_new, Phi_old, os_new, os_old):
    """The factored form of Eq. ic-tw: yhat_w = T yhat_{w-1} + c with
    T = Phi_w^T Phi_{w-1} [n_w][n_{w-1}] and c = Phi_w^T (os_{w-1} - os_w) ([n_w] or [n_w][B]),
    by plain matrix products (pinned against window_transition, P25)."""
    T = np.ascontiguousarray(Phi_new.T @ Phi_old)
    c = np.ascontiguousarray(Phi_new.T @ (os_old - os_new))
    return T, c


def rom_rk2avg_step(op, Yx, Yv, Ye, dt):
    """One hyper-reduced RK2-average step for every instance.  op: dict with keys
    base, closure_elems, closure_nodes, s0_nodes, sample_elems, Phi_x, Phi_v, Phi_e
    (closure rows), x_os, v_os, e_os, R_v, R_e, C_xv, c_x.  dt: [B].
    Returns (Yx1, Yv1, Ye1, dt_est[B])."""
    B = Yv.shape[1]
    dt = np.asarray(dt, dtype=np.float64)
    args = (op["base"], op["closure_elems"], op["closure_nodes"], op["s0_nodes"], op["sample_elems"])

    def forces(xS, vS, eS, wS):
        res = [sampled_force(*args, xS, vS, eS, wS, b) for b in range(B)]
        F1 = np.stack([r[0] for r in res], axis=1)
        FT = np.stack([r[1] for r in res], axis=1)
        dts = np.array([r[2] for r in res])
        return F1, FT, dts

    xS = lift(op["Phi_x"], op["x_os"], Yx)
    vS = lift(op["Phi_v"], op["v_os"], Yv)
    eS = lift(op["Phi_e"], op["e_os"], Ye)
    F1, _, dt1 = forces(xS, vS, eS, vS)
    Yv_h = Yv - 0.5 * dt * (op["R_v"] @ F1)
    vS_h = lift(op["Phi_v"], op["v_os"], Yv_h)
    _, FT, _ = forces(xS, vS, eS, vS_h)
    Ye_h = Ye + 0.5 * dt * (op["R_e"] @ FT)
    cx = op["c_x"][:, None] if op["c_x"].ndim == 1 else op["c_x"]   # [nx] or per instance [nx][B]
    Yx_h = Yx + 0.5 * dt * (cx + op["C_xv"] @ Yv_h)
    xS_h = lift(op["Phi_x"], op["x_os"], Yx_h)
    eS_h = lift(op["Phi_e"], op["e_os"], Ye_h)
    F1h, _, dt2 = forces(xS_h, vS_h, eS_h, vS_h)
    Yv1 = Yv - dt * (op["R_v"] @ F1h)
    Yvb = 0.5 * (Yv + Yv1)
    vS_b = lift(op["Phi_v"], op["v_os"], Yvb)
    _, FTh, _ = forces(xS_h, vS_h, eS_h, vS_b)
    Ye1 = Ye + dt * (op["R_e"] @ FTh)
    Yx1 = Yx + dt * (cx + op["C_xv"] @ Yvb)
    return Yx1, Yv1, Ye1, np.minimum(dt1, dt2)


def advance(op, Yx, Yv, Ye, t0, t_final, dt, beta1=0.85, beta2=1.02, gamma=0.8,
            max_iters=10**6, step=None):
    """Online time loop t0 -> t_final for every instance under the time-step controller of
    PAPER P:549-566, applied to each instance independently (each is its own simulation):
    all instances take one batched step with their own trial dt (0 once finished); an
    instance whose dt >= its estimate keeps its previous coordinates and retries with
    beta1 dt; an accepted one advances, growing dt by beta2 when dt <= gamma * estimate; the
    step that reaches t_final is shortened to land on it.  `step(Yx, Yv, Ye, dt[B]) ->
    (Yx1, Yv1, Ye1, dt_est[B])` defaults to rom_rk2avg_step(op, ...).
    Returns (Yx, Yv, Ye, t[B], next_dt[B], accepted[B], rejected[B], batched_steps)."""
    if step is None:
        def step(a, b_, c, h_):
            return rom_rk2avg_step(op, a, b_, c, h_)
    B = Yv.shape[1]
    t = np.full(B, float(t0))
    h = np.array(dt, dtype=np.float64).copy()
    ns = np.zeros(B, dtype=np.int64)
    nr = np.zeros(B, dtype=np.int64)
    it = 0
    while it < max_iters:
        act = t < t_final
        if not act.any():
            break
        htry = np.where(act, np.where(t_final - t < h, t_final - t, h), 0.0)
        Yx1, Yv1, Ye1, est = step(Yx, Yv, Ye, htry)
        it += 1
        keep = np.zeros(B, dtype=bool)
        for b in range(B):
            if htry[b] == 0.0:
                continue
            if np.isnan(est[b]) or htry[b] >= est[b]:   # invalid or too large (R26)
                h[b] = beta1 * htry[b]
                nr[b] += 1
                if nr[b] > 10000:
                    raise FloatingPointError(f"no admissible step found, instance {b}")
                continue
            keep[b] = True
            t[b] = t_final if htry[b] == t_final - t[b] else t[b] + htry[b]
            ns[b] += 1
            h[b] = beta2 * htry[b] if htry[b] <= gamma * est[b] else htry[b]
        Yx = np.where(keep[None, :], Yx1, Yx)
        Yv = np.where(keep[None, :], Yv1, Yv)
        Ye = np.where(keep[None, :], Ye1, Ye)
    return Yx, Yv, Ye, t, h, ns, nr, it


def window_transition(Phi_new, Phi_old, os_new, os_old, Y):
    """Initial reduced coordinates of time window w from those of window w-1, PAPER Eq.
    ic-tw, written out as the paper states it:
        yhat_w = Phi_w^T (os_{w-1} + Phi_{w-1} yhat_{w-1} - os_w)
    (lift with the old window's basis and offset, subtract the new offset, project on the new
    basis); offsets [rows] or [rows][B].  Evaluated as Phi_w^T (os_{w-1} - os_w) +
    Phi_w^T (Phi_{w-1} yhat): the offsets are differenced first (lifting and then
    subtracting a large offset would cancel catastrophically for the e field's spike).
    Independent of the factored T, c form (window_transition_ops; hydro_window_ops on the GPU)."""
    o2 = lambda a: a[:, None] if a.ndim == 1 else a   # [rows] -> [rows][1]
    d = o2(os_old) - o2(os_new)
    return Phi_new.T @ d + Phi_new.T @ (Phi_old @ Y)


def previous_window_offset(Phi_prev, os_prev, Y_prev):
    """The previous-window offset, PAPER Eq. previous_os, as written:
        os_w = os_{w-1} + Phi_{w-1} yhat_{w-1}(t_{w-1})
    (the lift of the previous window's final state; per instance, [rows][B])."""
    os2 = os_prev[:, None] if os_prev.ndim == 1 else os_prev
    return os2 + Phi_prev @ Y_prev


def window_transition_oblique(Phi_new, Phi_old, os_new, os_old, Y, M):
    """The M-oblique variant, PAPER Eq. ic2-tw, as written:
        yhat_w = (Phi_w^T M Phi_w)^{-1} Phi_w^T M (os_{w-1} + Phi_{w-1} yhat_{w-1} - os_w)
    with M the field's FOM mass matrix (M_V for velocity, M_E for energy; the position keeps
    Eq. ic-tw).  M: a function applying the mass matrix to a [N][k] array.  The offsets are
    differenced first, as in window_transition."""
    d = os_old - os_new
    d = d[:, None] if d.ndim == 1 else d
    Mhat = Phi_new.T @ M(Phi_new)
    rhs = Phi_new.T @ M(d) + Phi_new.T @ M(Phi_old @ Y)
    return np.linalg.solve(Mhat, rhs)


def windowed_advance(windows, Yx, Yv, Ye, t0, dt, beta1=0.85, beta2=1.02, gamma=0.8,
                     max_iters=10**6, offsets="fixed"):
    """The time-windowing online phase: for each window, `advance` with its
    own operators up to its end time, then map the reduced coordinates into the next
    window's bases (window_transition, from the two windows' bases and offsets in `op`).
    windows: list of dicts with keys op (the rom_rk2avg_step operators, incl. Phi_x/v/e and
    x_os/v_os/e_os) and t_end.  offsets = "previous": the offsets of window w > 1 are not
    taken from its op but formed at the transition by Eq. previous_os per
    instance, with c_x = Phi_x,w^T v_os,w per instance, and the new coordinates
    by Eq. ic-tw with those offsets (zero up to rounding).  Returns (Yx, Yv, Ye, t[B],
    next_dt[B], per-window (accepted, rejected))."""
    t = t0
    h = np.array(dt, dtype=np.float64)
    stats = []
    tB = None
    ops = [dict(w["op"]) for w in windows]
    for wi, w in enumerate(windows):
        Yx, Yv, Ye, tB, h, ns, nr, _ = advance(ops[wi], Yx, Yv, Ye, t, w["t_end"], h, beta1, beta2,
                                               gamma, max_iters)
        stats.append((ns, nr))
        t = w["t_end"]
        nxt = wi + 1
        if nxt < len(windows):
            o, n = ops[wi], ops[nxt]
            if offsets == "previous":
                n["x_os"] = previous_window_offset(o["Phi_x"], o["x_os"], Yx)
                n["v_os"] = previous_window_offset(o["Phi_v"], o["v_os"], Yv)
                n["e_os"] = previous_window_offset(o["Phi_e"], o["e_os"], Ye)
                n["c_x"] = n["Phi_x"].T @ n["v_os"]
            Yx = window_transition(n["Phi_x"], o["Phi_x"], n["x_os"], o["x_os"], Yx)
            Yv = window_transition(n["Phi_v"], o["Phi_v"], n["v_os"], o["v_os"], Yv)
            Ye = window_transition(n["Phi_e"], o["Phi_e"], n["e_os"], o["e_os"], Ye)
    return Yx, Yv, Ye, tB, h, stats


def indicator_term(f, Phi, M, U, Z):
    """One field of the Theorem-2 integrand (Eq. aposteriori-semi), as written:
        | (I - M Phi Mhat^{-1} Phi^T P) f |_2,   Mhat = Phi^T M Phi,
    with the DEIM projector P f = U (Z^T U)^+ Z^T f (numpy lstsq; the inverse when the
    sample count equals the basis size).  M: function applying the field's mass
    matrix to a [N][k] array."""
    Z = np.asarray(Z, dtype=np.int64)
    a = np.linalg.lstsq(U[Z], f[Z], rcond=None)[0]
    Pf = U @ a
    MPhi = M(Phi)
    Mhat = Phi.T @ MPhi
    z = np.linalg.solve(Mhat, Phi.T @ Pf)
    return float(np.linalg.norm(f - MPhi @ z))


def aposteriori_integrand(prob, x, v, e, Phi_v, Phi_e, U1, Z1, U2, Z2):
    """(eta_v, eta_e): the two Theorem-2 integrands at the state (x, v, e) -- the full-order
    F.1 and F^T.v (w = v) by the force oracle, M_V = I_dim (x) the scalar kinematic mass
    matrix (velocity dofs c * n_nodes + node), M_E the element blocks (DESIGN R29)."""
    from . import force as _f
    from . import fom as _fom
    m = prob.mesh
    out = _f(prob, x=x, v=v, e=e, w=v)
    F1 = np.asarray(out["F1"]).reshape(-1)
    FTv = np.asarray(out["FTw"]).reshape(-1)
    Mv, Me, n = _fom.mass_v(m), _fom.mass_e(m), m.n_nodes

    def MV(a):
        return np.concatenate([Mv @ a[c * n:(c + 1) * n] for c in range(m.dim)])

    def ME(a):
        return np.einsum("eij,ejk->eik", Me, a.reshape(m.n_elem, m.ne, -1)).reshape(a.shape)
    return (indicator_term(F1, Phi_v, MV, U1, Z1), indicator_term(FTv, Phi_e, ME, U2, Z2))

"""CPU oracle of the full-order RK2-average time step -- TEST INFRASTRUCTURE ONLY
(same import rules as oracle/__init__.py).

PAPER.md, Sec. 2 (semi-discrete FOM, Eq. fom P:403-411 and the RK2-average scheme
Eq. RK2-avg):

    M_V dv/dt = -F . 1,     M_E de/dt = F^T . v,     dx/dt = v

    v^{n+1/2} = v^n - (dt/2) M_V^{-1} F(U^n).1            e^{n+1/2} = e^n + (dt/2) M_E^{-1} F(U^n)^T v^{n+1/2}
    x^{n+1/2} = x^n + (dt/2) v^{n+1/2}
    v^{n+1}   = v^n - dt M_V^{-1} F(U^{n+1/2}).1         e^{n+1}   = e^n + dt M_E^{-1} F(U^{n+1/2})^T vbar
    x^{n+1}   = x^n + dt vbar,        vbar = (v^n + v^{n+1}) / 2

The mass matrices are constant in time (Lagrangian mass conservation):
    M_V[a][b] = sum_K sum_q w_q m_q phi_a(xi_q) phi_b(xi_q)      (per velocity component)
    M_E,K[i][j] = sum_q w_q m_q psi_i(xi_q) psi_j(xi_q)           (block diagonal)
with m_q = rho0_K detJ0(xi_q) (DESIGN R11).  The boundary condition v.n = 0
is imposed by removing the normal velocity components of boundary nodes from the
unknowns of M_V (they stay zero).  The discrete total energy
    E = 1/2 v^T M_V v + 1^T M_E e
is conserved exactly by the scheme (Proposition 7.1 of Dobrev et al.).

Plain definitions: tensor-product basis matrices built with np.kron, element matrices
assembled into a scipy.sparse matrix, linear solves by a sparse direct factorisation
(library primitives as steps), and the force by oracle.force.  Pins:
tests/test_fom_oracle_pins.py.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import force as _force
from . import tables as _tables


def basis(dim: int, k: int, q: int):
    """Tensor-product tables at the Gauss points (point q = q1 + Q q2 [+ Q^2 q3], node
    a = a1 + N a2 [+ N^2 a3], both first index fastest): values Phi [NQ][ND], reference
    gradients dPhi [dim][NQ][ND], L2 values Psi [NQ][NE], weights W [NQ]."""
    T = _tables(k, q)      # oracle.tables(k, q): the mpmath tables (the function, not the module)
    B = np.array(T["B"], dtype=np.float64)
    G = np.array(T["G"], dtype=np.float64)
    Bl = np.array(T["Bl"], dtype=np.float64)
    w = np.array(T["w"], dtype=np.float64)
    if dim == 2:
        Phi = np.kron(B, B)
        dPhi = np.stack([np.kron(B, G), np.kron(G, B)])
        Psi = np.kron(Bl, Bl)
        W = np.kron(w, w)
    else:
        Phi = np.kron(B, np.kron(B, B))
        dPhi = np.stack([np.kron(B, np.kron(B, G)), np.kron(B, np.kron(G, B)),
                         np.kron(G, np.kron(B, B))])
        Psi = np.kron(Bl, np.kron(Bl, Bl))
        W = np.kron(w, np.kron(w, w))
    return Phi, dPhi, Psi, W


def qp_mass(mesh) -> np.ndarray:
    """m_q = rho0_K detJ0(xi_q)  [E][NQ]  (density elimination)."""
    _, dPhi, _, _ = basis(mesh.dim, mesh.k, mesh.nq)
    X = mesh.x0[:, mesh.elem_nodes]                      # [d][E][ND]
    J = np.einsum("cea,dqa->eqcd", X, dPhi)              # J[e][q][c][d] = dx_c/dxi_d
    return mesh.rho0[:, None] * np.linalg.det(J)


def mass_v(mesh) -> sp.csr_matrix:
    """Scalar kinematic mass matrix [n_nodes][n_nodes] (the same block for every component)."""
    Phi, _, _, W = basis(mesh.dim, mesh.k, mesh.nq)
    m = qp_mass(mesh)
    Ke = np.einsum("qa,eq,qb->eab", Phi, m * W[None, :], Phi)   # [E][ND][ND]
    en = mesh.elem_nodes
    rows = np.repeat(en, en.shape[1], axis=1).ravel()
    cols = np.tile(en, (1, en.shape[1])).ravel()
    return sp.csr_matrix((Ke.ravel(), (rows, cols)), shape=(mesh.n_nodes, mesh.n_nodes))


def mass_e(mesh) -> np.ndarray:
    """Thermodynamic mass matrix blocks [E][NE][NE]."""
    _, _, Psi, W = basis(mesh.dim, mesh.k, mesh.nq)
    m = qp_mass(mesh)
    return np.einsum("qi,eq,qj->eij", Psi, m * W[None, :], Psi)


def bc_dofs_box(mesh) -> np.ndarray:
    """v.n = 0 on the box boundary: component c of every node on a face x_c = lo_c or
    hi_c (boundary nodes are never perturbed, DESIGN R17).  Sorted flat indices
    c*n_nodes + node."""
    out = []
    for c in range(mesh.dim):
        on = np.isclose(mesh.x0[c], mesh.lo[c]) | np.isclose(mesh.x0[c], mesh.hi[c])
        out.append(c * mesh.n_nodes + np.nonzero(on)[0])
    return np.sort(np.concatenate(out)).astype(np.int64)


class Fom:
    """Mass matrices, boundary dofs and factorisations of one mesh."""

    def __init__(self, mesh, bc: np.ndarray):
        self.mesh = mesh
        self.M = mass_v(mesh)
        self.ME = mass_e(mesh)
        self.bc = np.asarray(bc, dtype=np.int64)
        n, d = mesh.n_nodes, mesh.dim
        fixed = np.zeros(d * n, dtype=bool)
        fixed[self.bc] = True
        self.free = [np.nonzero(~fixed[c * n:(c + 1) * n])[0] for c in range(d)]
        self.lu = [spla.splu(self.M[f][:, f].tocsc()) for f in self.free]

    def solve_v(self, rhs: np.ndarray) -> np.ndarray:
        """M_V^{-1} rhs on the free dofs, zero on the constrained ones.  rhs [d][n]."""
        out = np.zeros_like(rhs)
        for c, (f, lu) in enumerate(zip(self.free, self.lu)):
            out[c, f] = lu.solve(rhs[c, f])
        return out

    def solve_e(self, rhs: np.ndarray) -> np.ndarray:
        return np.linalg.solve(self.ME, rhs[..., None])[..., 0]

    def energy(self, v: np.ndarray, e: np.ndarray):
        kin = 0.5 * sum(float(v[c] @ (self.M @ v[c])) for c in range(v.shape[0]))
        inte = float(np.einsum("eij,ej->", self.ME, e))
        return kin, inte


def rk2avg_step(fom: Fom, prob, x, v, e, dt: float, force=None):
    """One RK2-average step from (x, v, e); returns (x1, v1, e1, dt_est) with
    dt_est the minimum of the two stages' estimates.

    force(x, v, e, w) -> {"F1", "FTw", "dt", "status"} defaults to the corner force of
    oracle.force (w = None means w = v); the pins substitute closed-form force fields
    (tests/test_fom_oracle_pins.py P39-P41)."""
    if force is None:
        def force(x_, v_, e_, w_=None):
            return _force(prob, x=x_, v=v_, e=e_, w=w_)
    s1 = force(x, v, e)
    v_h = v - 0.5 * dt * fom.solve_v(s1["F1"])
    s1w = force(x, v, e, v_h)
    e_h = e + 0.5 * dt * fom.solve_e(s1w["FTw"])
    x_h = x + 0.5 * dt * v_h
    s2 = force(x_h, v_h, e_h)
    v1 = v - dt * fom.solve_v(s2["F1"])
    vbar = 0.5 * (v + v1)
    s2w = force(x_h, v_h, e_h, vbar)
    e1 = e + dt * fom.solve_e(s2w["FTw"])
    x1 = x + dt * vbar
    if s1["status"] or s2["status"]:   # tangled or non-finite stage: the step is invalid
        return x1, v1, e1, float("nan")
    return x1, v1, e1, min(s1["dt"], s2["dt"])


def advance(fom: Fom, prob, x, v, e, t0: float, t_final: float, dt: float, beta1=0.85,
            beta2=1.02, gamma=0.8, max_steps=10**6, step=None):
    """Time loop t0 -> t_final under the time-step controller of PAPER P:549-566:

      1. with dt and the state U^n, evaluate U^{n+1} and the estimate dt_est;
      2. if dt >= dt_est: dt <- beta1 dt and go to 1 (from U^n) -- also when the trial step
         is invalid (a stage tangles an element or its estimate is NaN, e.g. a negative
         energy, R12): dt_est = NaN then, read as "too large" (DESIGN R26);
      3. if dt <= gamma dt_est: dt <- beta2 dt;
      4. accept, n <- n + 1.

    The step that reaches t_final is shortened to land on it (reading: the paper runs to a
    final time t_f).  `step(x, v, e, dt) -> (x1, v1, e1, dt_est)` defaults to
    rk2avg_step on (fom, prob).  Returns (x, v, e, t, next_dt, accepted, rejected)."""
    if step is None:
        def step(x_, v_, e_, h_):
            return rk2avg_step(fom, prob, x_, v_, e_, h_)
    t, h, ns, nr = t0, dt, 0, 0
    while t < t_final and ns < max_steps:
        h_try = t_final - t if t_final - t < h else h
        x1, v1, e1, est = step(x, v, e, h_try)
        if np.isnan(est) or h_try >= est:
            h = beta1 * h_try
            nr += 1
            if nr > 10000:
                raise FloatingPointError("no admissible step found")
            continue
        x, v, e = x1, v1, e1
        t = t_final if h_try == t_final - t else t + h_try
        ns += 1
        h = beta2 * h_try if h_try <= gamma * est else h_try
    return x, v, e, t, h, ns, nr

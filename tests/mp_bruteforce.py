"""Brute-force 40-digit evaluation of the force definition (pin P11).

Independent of `oracle/` (it does not import it) and of the CUDA path: basis
functions are evaluated directly as Lagrange products on closed-form nodes,
quadrature points come from mpmath root finding, eigenvalues from mpmath.eigsy,
inverses/determinants from mpmath matrices.  Only used on 1-4 element meshes.

Definition (DESIGN R1-R3, R11; PAPER Eq. fom, Eq. EOS P:374-376,
Eq. adaptive-timestep):
  F1[(a,c)] = sum_K sum_q w_q detJ (sigma J^-T gradhat phi_a)_c
  FTw[K,j]  = sum_q w_q detJ psi_j (sigma : grad w)
  dt        = min_q alpha / (cs/h + alpha_mu mu / (rho h^2))
"""
from __future__ import annotations

import mpmath as mp

mp.mp.dps = 40


def gll_nodes(k):
    if k == 1:
        return [mp.mpf(0), mp.mpf(1)]
    if k == 2:
        return [mp.mpf(0), mp.mpf(1) / 2, mp.mpf(1)]
    if k == 3:
        s5 = mp.sqrt(5)
        return [mp.mpf(0), (5 - s5) / 10, (5 + s5) / 10, mp.mpf(1)]
    raise ValueError(k)


def gl_rule(q):
    """Gauss-Legendre on [0,1] from the roots of the Legendre polynomial coefficients."""
    coeffs = mp.taylor(lambda t: mp.legendre(q, t), 0, q)[::-1]
    roots = sorted(mp.re(r) for r in mp.polyroots(coeffs, maxsteps=200, extraprec=200))
    pts, wts = [], []
    for r in roots:
        dp = mp.diff(lambda t: mp.legendre(q, t), r)
        wts.append(1 / ((1 - r * r) * dp * dp))
        pts.append((r + 1) / 2)
    return pts, wts


def lag(nodes, j, t):
    v = mp.mpf(1)
    for m, xm in enumerate(nodes):
        if m != j:
            v *= (t - xm) / (nodes[j] - xm)
    return v


def dlag(nodes, j, t):
    return mp.diff(lambda s: lag(nodes, j, s), t)


def evaluate(prob, elems=None):
    """Returns dict(F1 [d][n_nodes] (mp), FTw {K: [ne]}, dt) for `prob`."""
    m = prob.mesh
    dim, k, q = m.dim, m.k, m.nq
    n = k + 1
    gll = gll_nodes(k)
    gl_l2, _ = gl_rule(k)
    xi, wq = gl_rule(q)
    B = [[lag(gll, a, t) for a in range(n)] for t in xi]
    G = [[dlag(gll, a, t) for a in range(n)] for t in xi]
    Bl = [[lag(gl_l2, j, t) for j in range(k)] for t in xi]
    elems = range(m.n_elem) if elems is None else elems
    F1 = [[mp.mpf(0)] * m.n_nodes for _ in range(dim)]
    FTw = {}
    dt = mp.inf
    nd, ne = n ** dim, k ** dim
    qps = [(i, j) for j in range(q) for i in range(q)] if dim == 2 else \
          [(i, j, l) for l in range(q) for j in range(q) for i in range(q)]
    loc = [(i, j) for j in range(n) for i in range(n)] if dim == 2 else \
          [(i, j, l) for l in range(n) for j in range(n) for i in range(n)]
    locl2 = [(i, j) for j in range(k) for i in range(k)] if dim == 2 else \
            [(i, j, l) for l in range(k) for j in range(k) for i in range(k)]
    w_vec = prob.v if prob.w is None else prob.w
    for K in elems:
        en = [int(t) for t in m.elem_nodes[K]]
        X = [[mp.mpf(float(prob.x[c][en[a]])) for a in range(nd)] for c in range(dim)]
        X0 = [[mp.mpf(float(m.x0[c][en[a]])) for a in range(nd)] for c in range(dim)]
        V = [[mp.mpf(float(prob.v[c][en[a]])) for a in range(nd)] for c in range(dim)]
        W = [[mp.mpf(float(w_vec[c][en[a]])) for a in range(nd)] for c in range(dim)]
        Ek = [mp.mpf(float(t)) for t in prob.e[K]]
        gam = mp.mpf(float(prob.gamma[K]))
        rho0 = mp.mpf(float(m.rho0[K]))
        F1K = [[mp.mpf(0)] * dim for _ in range(nd)]
        FK = [mp.mpf(0)] * ne
        for qi in qps:
            # gradhat phi_a at this qp
            Dphi = []
            for la in loc:
                row = []
                for dlt in range(dim):
                    v = mp.mpf(1)
                    for dd in range(dim):
                        v *= (G if dd == dlt else B)[qi[dd]][la[dd]]
                    row.append(v)
                Dphi.append(row)
            psi = []
            for lj in locl2:
                v = mp.mpf(1)
                for dd in range(dim):
                    v *= Bl[qi[dd]][lj[dd]]
                psi.append(v)
            wqp = mp.mpf(1)
            for dd in range(dim):
                wqp *= wq[qi[dd]]
            def grad(F):
                return mp.matrix([[mp.fsum(F[c][a] * Dphi[a][d] for a in range(nd))
                                   for d in range(dim)] for c in range(dim)])
            J, J0, Gv, Gw = grad(X), grad(X0), grad(V), grad(W)
            det, det0 = mp.det(J), mp.det(J0)
            Ji = J ** -1
            rho = rho0 * det0 / det
            eq = mp.fsum(psi[j] * Ek[j] for j in range(ne))
            p = (gam - 1) * rho * eq
            cs = mp.sqrt(max(gam * (gam - 1) * eq, 0))
            h = mp.sqrt(min(mp.eigsy(J.T * J, eigvals_only=True)))
            gv = Gv * Ji
            eps = (gv + gv.T) / 2
            if prob.visc:
                lam = min(mp.eigsy(eps, eigvals_only=True))
                mu = rho * h * (prob.q1 * cs + prob.q2 * h * (-min(lam, 0)))
            else:
                mu = mp.mpf(0)
            dtq = prob.alpha / (cs / h + prob.alpha_mu * mu / (rho * h * h))
            dt = min(dt, dtq)
            sig = mu * eps - p * mp.eye(dim)
            S = wqp * det * sig * Ji.T
            for a in range(nd):
                for c in range(dim):
                    F1K[a][c] += mp.fsum(S[c, d] * Dphi[a][d] for d in range(dim))
            gw = Gw  # reference gradient of w
            A = mp.fsum(S[c, d] * gw[c, d] for c in range(dim) for d in range(dim))
            for j in range(ne):
                FK[j] += psi[j] * A
        for a in range(nd):
            for c in range(dim):
                F1[c][en[a]] += F1K[a][c]
        FTw[K] = FK
    return dict(F1=F1, FTw=FTw, dt=dt)

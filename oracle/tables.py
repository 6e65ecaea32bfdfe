"""Oracle-side 1D basis and quadrature tables (TEST INFRASTRUCTURE ONLY).

Computed here with mpmath at 50 significant digits and rounded once to the
nearest double. The CUDA library computes its own tables independently (binary128
Newton in csrc/tables.cpp); both are correctly rounded, so a test can demand the
two sets agree bit for bit -- no table or generator is shared.

Readings (R5, R6; PAPER P:384-394 defers the basis to Dobrev 2012):
  * reference element [0,1]^d;
  * quadrature: tensor Gauss-Legendre with q points per dimension;
  * H1 (kinematic) basis: degree-k Lagrange polynomials on the k+1 Gauss-Lobatto
    points {0, roots of P_k', 1};
  * L2 (thermodynamic) basis: degree-(k-1) Lagrange polynomials on the k
    Gauss-Legendre points.
Tables:  xi[q], w[q];  B[q][a] = l_a(xi_q), G[q][a] = l_a'(xi_q)  (a < k+1);
         Bl[q][j] = lGL_j(xi_q)  (j < k).
"""
from __future__ import annotations

import functools

import mpmath

_DPS = 50


def _legendre_roots(n: int):
    """Roots of P_n on [-1,1], ascending, and Gauss weights."""
    with mpmath.workdps(_DPS + 10):
        xs, ws = [], []
        for i in range(n):
            # Chebyshev-like initial guess, Newton on P_n
            x = -mpmath.cos(mpmath.pi * (i + mpmath.mpf(3) / 4) / (n + mpmath.mpf(1) / 2))
            for _ in range(100):
                p = mpmath.legendre(n, x)
                dp = n * (x * p - mpmath.legendre(n - 1, x)) / (x * x - 1)
                dx = p / dp
                x -= dx
                if abs(dx) < mpmath.mpf(10) ** (-(_DPS + 5)):
                    break
            p1 = mpmath.legendre(n - 1, x)
            dp = n * (x * mpmath.legendre(n, x) - p1) / (x * x - 1)
            xs.append(x)
            ws.append(2 / ((1 - x * x) * dp * dp))
        order = sorted(range(n), key=lambda i: xs[i])
        return [xs[i] for i in order], [ws[i] for i in order]


def _lobatto_nodes(k: int):
    """k+1 Gauss-Lobatto points on [-1,1]: -1, roots of P_k', 1."""
    with mpmath.workdps(_DPS + 10):
        if k == 1:
            return [mpmath.mpf(-1), mpmath.mpf(1)]
        inner = []
        for i in range(1, k):
            x = -mpmath.cos(mpmath.pi * i / k)
            dP = lambda t: mpmath.diff(lambda s: mpmath.legendre(k, s), t)
            x = mpmath.findroot(dP, x, tol=mpmath.mpf(10) ** (-(_DPS + 5)))
            inner.append(x)
        return [mpmath.mpf(-1)] + sorted(inner) + [mpmath.mpf(1)]


def _lagrange(nodes, j, t):
    v = mpmath.mpf(1)
    for m, xm in enumerate(nodes):
        if m != j:
            v *= (t - xm) / (nodes[j] - xm)
    return v


def _lagrange_d(nodes, j, t):
    s = mpmath.mpf(0)
    for i, xi in enumerate(nodes):
        if i == j:
            continue
        term = 1 / (nodes[j] - xi)
        for m, xm in enumerate(nodes):
            if m != j and m != i:
                term *= (t - xm) / (nodes[j] - xm)
        s += term
    return s


def _to_double(x) -> float:
    # mpmath's float() rounds to nearest from its binary representation
    return float(mpmath.mpf(x))


@functools.lru_cache(maxsize=None)
def tables_mp(k: int, q: int):
    """High-precision tables on [0,1] (mpmath values)."""
    with mpmath.workdps(_DPS + 10):
        g, w = _legendre_roots(q)
        xi = [(x + 1) / 2 for x in g]
        wq = [wi / 2 for wi in w]
        gll = [(x + 1) / 2 for x in _lobatto_nodes(k)]
        gl_l2 = [(x + 1) / 2 for x in _legendre_roots(k)[0]]
        B = [[_lagrange(gll, a, t) for a in range(k + 1)] for t in xi]
        G = [[_lagrange_d(gll, a, t) for a in range(k + 1)] for t in xi]
        Bl = [[_lagrange(gl_l2, j, t) for j in range(k)] for t in xi]
        return dict(xi=xi, w=wq, gll=gll, gl_l2=gl_l2, B=B, G=G, Bl=Bl)


@functools.lru_cache(maxsize=None)
def tables(k: int, q: int):
    """Correctly rounded double tables (python floats, nested lists)."""
    t = tables_mp(k, q)
    cv = lambda a: [_to_double(v) for v in a]
    return dict(xi=cv(t["xi"]), w=cv(t["w"]), gll=cv(t["gll"]), gl_l2=cv(t["gl_l2"]),
                B=[cv(r) for r in t["B"]], G=[cv(r) for r in t["G"]], Bl=[cv(r) for r in t["Bl"]])

"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the pin of DESIGN.md "Oracle pins" (P1..P14) it implements and
is chosen so that a plausible mistake (a dropped term, a wrong sign or index, a
transposed operand) fails at least one of them.
"""
from __future__ import annotations

import json
import math
import os

import mpmath
import numpy as np
import pytest

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# --------------------------------------------------------------------------- tables (P10)
@pytest.mark.parametrize("k,q", [(2, 4), (3, 6), (1, 2)])
def test_tables_polynomial_exactness(oracle_lib, k, q):
    """P10: GL rule integrates x^j exactly for j <= 2q-1; B, G, Bl reproduce
    polynomials of their degree and their derivatives (Lagrange property)."""
    T = oracle_lib.tables(k, q)
    xi, w = np.array(T["xi"]), np.array(T["w"])
    assert abs(w.sum() - 1.0) < 4e-16
    for j in range(2 * q):
        assert abs((w * xi ** j).sum() - 1.0 / (j + 1)) < 2e-15, j
    gll, gl2 = np.array(T["gll"]), np.array(T["gl_l2"])
    B, G, Bl = np.array(T["B"]), np.array(T["G"]), np.array(T["Bl"])
    assert B.shape == (q, k + 1) and Bl.shape == (q, k)
    for p in range(k + 1):
        assert np.allclose(B @ gll ** p, xi ** p, atol=2e-15, rtol=0)
        dp = p * xi ** (p - 1) if p > 0 else np.zeros(q)
        assert np.allclose(G @ gll ** p, dp, atol=2e-14, rtol=0)
    for p in range(k):
        assert np.allclose(Bl @ gl2 ** p, xi ** p, atol=2e-15, rtol=0)
    # partition of unity / zero-sum derivative rows
    assert np.abs(B.sum(axis=1) - 1).max() <= 4 * 2.0 ** -52
    assert np.abs(G.sum(axis=1)).max() <= 32 * 2.0 ** -52 * np.abs(G).max()


def test_tables_closed_forms(oracle_lib):
    """P10: closed-form nodes and the GLL basis integrals (tests/golden gll_integrals)."""
    T2 = oracle_lib.tables(2, 4)
    r = [math.sqrt(3 / 7 - 2 / 7 * math.sqrt(6 / 5)), math.sqrt(3 / 7 + 2 / 7 * math.sqrt(6 / 5))]
    ref = sorted([(1 - r[1]) / 2, (1 - r[0]) / 2, (1 + r[0]) / 2, (1 + r[1]) / 2])
    assert np.allclose(T2["xi"], ref, rtol=0, atol=3e-16)
    wref = [(18 - math.sqrt(30)) / 72, (18 + math.sqrt(30)) / 72] * 1
    assert np.allclose(T2["w"], [wref[0], wref[1], wref[1], wref[0]], rtol=0, atol=3e-16)
    assert T2["gll"] == [0.0, 0.5, 1.0]
    g = 1 / math.sqrt(3)
    assert np.allclose(T2["gl_l2"], [(1 - g) / 2, (1 + g) / 2], rtol=0, atol=3e-16)
    T3 = oracle_lib.tables(3, 6)
    s5 = math.sqrt(5)
    assert np.allclose(T3["gll"], [0, (5 - s5) / 10, (5 + s5) / 10, 1], rtol=0, atol=3e-16)
    assert np.allclose(T3["gl_l2"], [(1 - math.sqrt(0.6)) / 2, 0.5, (1 + math.sqrt(0.6)) / 2],
                       rtol=0, atol=3e-16)
    for k, q in ((2, 4), (3, 6)):
        T = oracle_lib.tables(k, q)
        integ = np.array(T["w"]) @ np.array(T["B"])
        assert np.allclose(integ, GOLD["gll_integrals"][str(k)], rtol=0, atol=2e-16)


@pytest.mark.parametrize("k,q", [(2, 4), (3, 6)])
def test_tables_correctly_rounded(oracle_lib, k, q):
    """P10: every table entry is the double nearest to a 60-digit value, rounded
    through a decimal string (independent of mpmath's float conversion)."""
    import importlib
    ot = importlib.import_module("oracle.tables")
    mp_t = ot.tables_mp(k, q)
    T = oracle_lib.tables(k, q)
    for key in ("xi", "w"):
        for a, b in zip(T[key], mp_t[key]):
            assert a == float(mpmath.nstr(b, 40, strip_zeros=False))
    for key in ("B", "G", "Bl"):
        for ra, rb in zip(T[key], mp_t[key]):
            for a, b in zip(ra, rb):
                assert a == float(mpmath.nstr(b, 40, strip_zeros=False))


# --------------------------------------------------------------------------- lmin3, det (P8)
def _sym(a6):
    a = np.array([[a6[0], a6[3], a6[4]], [a6[3], a6[1], a6[5]], [a6[4], a6[5], a6[2]]])
    return a


def test_lmin3_vs_eigvalsh(oracle_lib):
    """P8: the contract's lmin3 (DESIGN A.4 / R30: closed form + two Newton steps, Jacobi
    near a double smallest eigenvalue) vs LAPACK on random, near-double-root, near-isotropic
    and graded matrices: |err| <= 4e-15 * ||A||."""
    rng = np.random.default_rng(7)
    worst = 0.0
    for i in range(3000):
        kind = i % 4
        if kind == 0:
            a = rng.standard_normal(6)
        elif kind == 1:      # near double root
            Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            lam = np.array([1.0, 1.0 + 1e-9 * rng.standard_normal(), -2.0 + rng.standard_normal()])
            M = Q @ np.diag(lam) @ Q.T
            a = [M[0, 0], M[1, 1], M[2, 2], M[0, 1], M[0, 2], M[1, 2]]
        elif kind == 2:      # near-isotropic J^T J
            J = np.eye(3) * 0.01875 + 1e-4 * rng.standard_normal((3, 3))
            M = J.T @ J
            a = [M[0, 0], M[1, 1], M[2, 2], M[0, 1], M[0, 2], M[1, 2]]
        else:                # graded scales
            a = rng.standard_normal(6) * 10.0 ** rng.integers(-8, 8)
        A = _sym(a)
        ref = np.linalg.eigvalsh(A)[0]
        got = oracle_lib.lmin3(a)
        err = abs(got - ref) / np.abs(A).max()
        worst = max(worst, err)
    assert worst < 4e-15, worst


@pytest.mark.parametrize("gap_lo,gap_hi,third", [(-14, -4, 3.0), (-4, -1, 3.0), (-14, -1, -2.0)])
def test_lmin3_double_root_and_branch_boundary(oracle_lib, gap_lo, gap_hi, third):
    """P8 (R30): eigenvalues (1, 1 + d, third) in a random frame, d log-uniform.  With
    third = 3 the smallest eigenvalue is (nearly) double: d < ~1e-4 lands in the Jacobi
    branch (r > 1 - 2^-13), larger d in the closed form right at its boundary, where the
    Newton root's conditioning is worst (f'(c) >= sqrt(24 * 2^-13) = 0.054, i.e. an error
    of at most ~20x the closed form's rounding level); third = -2 makes the smallest
    eigenvalue simple and the top pair double (r near -1, well conditioned).  Bound:
    5e-14 ||A|| (measured worst 1.1e-14 over 2e4 such matrices)."""
    rng = np.random.default_rng(int(-gap_lo * 10 + third))
    worst = 0.0
    for _ in range(2000):
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        d = 10.0 ** rng.uniform(gap_lo, gap_hi)
        M = Q @ np.diag([1.0, 1.0 + d, third]) @ Q.T
        a = [M[0, 0], M[1, 1], M[2, 2], M[0, 1], M[0, 2], M[1, 2]]
        ref = np.linalg.eigvalsh(_sym(a))[0]
        worst = max(worst, abs(oracle_lib.lmin3(a) - ref) / np.abs(M).max())
    assert worst < 5e-14, worst


def test_lmin3_branches_taken(oracle_lib):
    """Both branches of R30 are exercised by the force evaluation of a C2-shaped mesh (the
    instrumented counters of the oracle): most points take the closed form, a few the Jacobi
    fallback."""
    import workloads as W
    oracle_lib.force(W.small("c2"))      # flushes counts of earlier direct lmin3 calls
    oracle_lib.lmin3_fallback_stats(reset=True)
    oracle_lib.force(W.small("c2"))
    rot, calls, fb = oracle_lib.lmin3_fallback_stats(reset=True)
    assert calls > 0 and 0 <= fb < 0.05 * calls


def test_lmin3_special_cases(oracle_lib):
    """P8: diagonal, zero, isotropic exact; exactly degenerate diagonal with tiny
    off-diagonals (the 0/0 hazard of a bare a_pq == 0 test) stays finite."""
    assert oracle_lib.lmin3([3.0, -2.0, 5.0, 0, 0, 0]) == -2.0
    assert oracle_lib.lmin3([0.0] * 6) == 0.0
    assert oracle_lib.lmin3([0.25] * 3 + [0.0] * 3) == 0.25
    a = [0.25, 0.25, 0.0625, 1e-17, -3e-17, 2e-17]
    r = oracle_lib.lmin3(a)
    assert math.isfinite(r) and abs(r - np.linalg.eigvalsh(_sym(a))[0]) < 1e-17
    # 2x2 block with exact equal diagonal: eigenvalues d +- |b|
    assert abs(oracle_lib.lmin3([1.0, 1.0, 4.0, 0.5, 0.0, 0.0]) - 0.5) < 4e-16


def test_det_vs_numpy(oracle_lib):
    rng = np.random.default_rng(3)
    for _ in range(200):
        J = rng.standard_normal((3, 3))
        assert abs(oracle_lib.det(3, J) - np.linalg.det(J)) < 1e-14 * max(1, abs(np.linalg.det(J)))
        J2 = rng.standard_normal((2, 2))
        assert abs(oracle_lib.det(2, J2) - np.linalg.det(J2)) < 1e-14


# --------------------------------------------------------------------------- single-element closed forms
def _affine_element(dim, k, nq, A, e_val=2.0, gamma=1.4, visc=True):
    """One element: the reference lattice of [0,1]^d mapped by x = A xi."""
    mesh = W.lattice_mesh(dim, k, nq, (1,) * dim, (0.0,) * dim, (1.0,) * dim)
    mesh.x0 = np.ascontiguousarray(np.asarray(A) @ mesh.x0)
    e = np.full((1, mesh.ne), e_val)
    return W.Problem("affine", mesh, mesh.x0.copy(), np.zeros_like(mesh.x0), e,
                     np.array([gamma]), visc=visc)


def _ref_face_integrals(dim, k, gll_w):
    """D[a][delta] = int_ref d_delta phi_a = (delta_{a_d=n-1} - delta_{a_d=0}) prod_{d'!=d} w[a_d']."""
    n = k + 1
    loc = [(i, j) for j in range(n) for i in range(n)] if dim == 2 else \
          [(i, j, l) for l in range(n) for j in range(n) for i in range(n)]
    D = np.zeros((len(loc), dim))
    for a, la in enumerate(loc):
        for d in range(dim):
            s = (1.0 if la[d] == n - 1 else 0.0) - (1.0 if la[d] == 0 else 0.0)
            for dd in range(dim):
                if dd != d:
                    s *= gll_w[la[dd]]
            D[a, d] = s
    return D


@pytest.mark.parametrize("dim,k,nq", [(2, 2, 4), (3, 2, 4), (2, 3, 6), (3, 3, 6)])
def test_P1_uniform_pressure_affine(oracle_lib, dim, k, nq):
    """P1: single affine element, uniform p, v = 0:
    (F.1)_{a,c} = -p detA sum_delta A^-T[c][delta] int_ref d_delta phi_a (face integrals
    with GLL weights), and F^T.v == 0 exactly (P5)."""
    rng = np.random.default_rng(dim * 10 + k)
    A = np.diag(rng.uniform(0.5, 2.0, dim)) + 0.2 * rng.standard_normal((dim, dim))
    prob = _affine_element(dim, k, nq, A)
    r = oracle_lib.force(prob)
    assert r["status"] == 0
    p = (1.4 - 1.0) * 1.0 * 2.0
    D = _ref_face_integrals(dim, k, GOLD["gll_integrals"][str(k)])
    ref = -p * np.linalg.det(A) * (np.linalg.inv(A).T @ D.T)      # [c][a]
    got = r["F1"][:, prob.mesh.elem_nodes[0]]
    assert np.abs(got - ref).max() < 2e-14 * np.abs(ref).max()
    assert np.all(r["FTw"] == 0.0)
    # centre node of a Q2 element carries no force
    if k == 2:
        centre = prob.mesh.elem_nodes[0][(k + 1) ** dim // 2]
        assert np.abs(r["F1"][:, centre]).max() < 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("dim,k,nq", [(2, 2, 4), (3, 2, 4), (3, 3, 6)])
def test_P3_linear_velocity_affine(oracle_lib, dim, k, nq):
    """P3: affine element, v = G x + b, uniform e: constant sigma computed here with
    numpy (eigvalsh, svd):  F.1 = sigma-weighted face integrals and
    (F^T v)_j = (sigma : G) |K| prod GL weights; dt by its formula (P9)."""
    rng = np.random.default_rng(100 + dim * 10 + k)
    A = np.diag(rng.uniform(0.5, 1.5, dim)) + 0.15 * rng.standard_normal((dim, dim))
    Gm = 0.3 * rng.standard_normal((dim, dim))
    b = rng.standard_normal(dim)
    prob = _affine_element(dim, k, nq, A, e_val=1.7, gamma=5.0 / 3.0)
    prob.v = np.ascontiguousarray(Gm @ prob.x + b[:, None])
    r = oracle_lib.force(prob)
    gam, e = 5.0 / 3.0, 1.7
    rho = 1.0
    p = (gam - 1) * rho * e
    cs = math.sqrt(gam * (gam - 1) * e)
    h = np.linalg.svd(A, compute_uv=False).min()
    eps = 0.5 * (Gm + Gm.T)
    lam = np.linalg.eigvalsh(eps)[0]
    mu = rho * h * (0.5 * cs + 2.0 * h * (-min(lam, 0.0)))
    sig = mu * eps - p * np.eye(dim)
    D = _ref_face_integrals(dim, k, GOLD["gll_integrals"][str(k)])
    detA = np.linalg.det(A)
    ref = detA * (sig @ np.linalg.inv(A).T @ D.T)
    got = r["F1"][:, prob.mesh.elem_nodes[0]]
    assert np.abs(got - ref).max() < 1e-13 * np.abs(ref).max()
    wgl = np.polynomial.legendre.leggauss(k)[1] / 2.0
    if dim == 2:
        wj = np.outer(wgl, wgl).ravel()
    else:
        wj = np.einsum("i,j,k->ijk", wgl, wgl, wgl).ravel()
    ref_ftv = (sig * Gm).sum() * detA * wj
    scale = (np.abs(sig) * np.abs(Gm)).sum() * abs(detA) * wj.max()
    assert np.abs(r["FTw"][0] - ref_ftv).max() < 1e-13 * scale
    dt = 0.5 / (cs / h + 2.5 * mu / (rho * h * h))
    assert abs(r["dt"] - dt) < 1e-14 * dt


def test_P9_eos_and_dt_worked_values(oracle_lib):
    """P9: SPEC worked values through the oracle. A unit square element (h = 1 by
    R2) with e = p/((gamma-1) rho) and v = 0, inviscid: the dt formula with mu = 0
    gives alpha h / cs; doubling alpha doubles dt exactly."""
    for rho, e, gam, p in GOLD["eos_examples"]["cases"]:
        assert abs((gam - 1.0) * rho * e - p) < 1e-15
    d = GOLD["dt_example"]
    assert d["alpha"] / (d["cs"] / d["h"]) == d["dt"]
    # through the oracle: choose e so that cs = 1 on an element of width 0.5
    gam = 1.4
    e = 1.0 / (gam * (gam - 1.0))
    prob = _affine_element(2, 2, 4, np.diag([0.5, 0.5]), e_val=e, gamma=gam, visc=False)
    r = oracle_lib.force(prob, mode=1)
    cs = math.sqrt(gam * (gam - 1.0) * e)
    assert abs(r["dt"] - 0.5 * 0.5 / cs) < 1e-15
    prob.alpha = 1.0
    assert oracle_lib.force(prob, mode=1)["dt"] == 2 * r["dt"]


# --------------------------------------------------------------------------- multi-element pins
@pytest.mark.parametrize("name", ["c0", "c2", "c3", "tg"])
def test_P2_interior_equilibrium(oracle_lib, name):
    """P2: uniform rho0, e, gamma, x = x0 (curved, perturbed), v = 0 => F.1 = 0 at
    every interior node up to rounding (exact GL quadrature, R6)."""
    prob = W.small(name)
    prob.v = np.zeros_like(prob.v)
    prob.e = np.full_like(prob.e, 1.3)
    prob.gamma = np.full_like(prob.gamma, 1.4)
    prob.mesh.rho0 = np.ones_like(prob.mesh.rho0)
    r = oracle_lib.force(prob)
    inner = ~W.boundary_nodes(prob.mesh)
    rel = np.abs(r["F1"][:, inner]) / r["F1mag"][:, inner]
    assert rel.max() < 1e-13
    bnd = W.boundary_nodes(prob.mesh)
    assert np.abs(r["F1"][:, bnd]).max() > 1e-6      # boundary nodes carry the wall force


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "tg"])
def test_P4_energy_identity(oracle_lib, name):
    """P4: v^T (F.1) = 1^T (F^T v) (underpins P:506-508)."""
    prob = W.small(name)
    r = oracle_lib.force(prob)
    lhs = (prob.v * r["F1"]).sum()
    rhs = r["FTw"].sum()
    scale = (np.abs(prob.v) * r["F1mag"]).sum() + r["FTwmag"].sum()
    assert abs(lhs - rhs) <= 1e-13 * scale


def test_P4_energy_identity_w_not_v(oracle_lib):
    """P4 with w != v (RK2-average stage): w^T (F.1) = 1^T (F^T w)."""
    prob = W.small("c2")
    rng = np.random.default_rng(5)
    prob.w = np.ascontiguousarray(prob.v + 0.1 * rng.standard_normal(prob.v.shape))
    r = oracle_lib.force(prob)
    lhs = (prob.w * r["F1"]).sum()
    scale = (np.abs(prob.w) * r["F1mag"]).sum() + r["FTwmag"].sum()
    assert abs(lhs - r["FTw"].sum()) <= 1e-13 * scale


def test_P5_zero_velocity(oracle_lib):
    """P5: F^T v == 0 bitwise at v = 0."""
    prob = W.small("c2")
    prob.v = np.zeros_like(prob.v)
    r = oracle_lib.force(prob)
    assert np.all(r["FTw"] == 0.0)


@pytest.mark.parametrize("name", ["c0", "c2", "c3"])
def test_P6_power_of_two_scaling(oracle_lib, name):
    """P6: x, x0 -> 2x, 2x0 => F.1 and F^T v scale by 2^(d-1), dt by 2, bitwise."""
    prob = W.small(name)
    r1 = oracle_lib.force(prob)
    d = prob.mesh.dim
    prob.mesh.x0 = prob.mesh.x0 * 2.0
    prob.x = prob.x * 2.0
    r2 = oracle_lib.force(prob)
    assert np.array_equal(r2["F1"], r1["F1"] * 2.0 ** (d - 1))
    assert np.array_equal(r2["FTw"], r1["FTw"] * 2.0 ** (d - 1))
    assert r2["dt"] == 2.0 * r1["dt"]


def test_P7_translation_rotation(oracle_lib):
    """P7: translation leaves F unchanged; a rotation R maps F.1 -> R F.1 per node
    and leaves F^T v and dt unchanged (within tolerance)."""
    prob = W.small("c2")
    r0 = oracle_lib.force(prob)
    tol = 1e-12
    # translation
    c = np.array([[0.3], [-0.2], [0.7]])
    pt = W.small("c2")
    pt.mesh.x0 = pt.mesh.x0 + c
    pt.x = pt.x + c
    rt = oracle_lib.force(pt)
    assert np.abs(rt["F1"] - r0["F1"]).max() < tol * np.abs(r0["F1mag"]).max()
    assert abs(rt["dt"] - r0["dt"]) < 1e-12 * r0["dt"]
    # rotation
    th = 0.7
    R = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1.0]])
    R = R @ np.array([[1, 0, 0], [0, math.cos(0.3), -math.sin(0.3)], [0, math.sin(0.3), math.cos(0.3)]])
    pr = W.small("c2")
    pr.mesh.x0 = np.ascontiguousarray(R @ pr.mesh.x0)
    pr.x = np.ascontiguousarray(R @ pr.x)
    pr.v = np.ascontiguousarray(R @ pr.v)
    rr = oracle_lib.force(pr)
    assert np.abs(rr["F1"] - R @ r0["F1"]).max() < tol * r0["F1mag"].max()
    assert np.abs(rr["FTw"] - r0["FTw"]).max() < tol * r0["FTwmag"].max()
    assert abs(rr["dt"] - r0["dt"]) < 1e-12 * r0["dt"]


def test_tangled_and_nan(oracle_lib):
    """Failure detection: the lowest element with detJ <= 0 is reported; NaN energy
    gives NaN dt (DESIGN R15, R16)."""
    prob = W.small("c2")
    m = prob.mesh
    # fold element 7 and 40: move their centre node far outside
    for K in (40, 7):
        centre = m.elem_nodes[K][13]
        prob.x[0, centre] += 5 * m.h[0]
    r = oracle_lib.force(prob, mode=1)
    assert r["status"] == 4 and r["first_bad"] == 7
    prob = W.small("c2")
    prob.e[3, 2] = np.nan
    r = oracle_lib.force(prob, mode=1)
    assert r["status"] == 5 and math.isnan(r["dt"])


def test_elist_restriction_matches_full(oracle_lib):
    """The element-list mode (used for sampled parity) equals the full evaluation on
    nodes whose every element is listed."""
    prob = W.small("c2")
    full = oracle_lib.force(prob)
    sample = np.array([3, 17, 50, 51], dtype=np.int32)
    cl = W.vertex_closure(prob.mesh, sample)
    part = oracle_lib.force(prob, elist=cl)
    nodes = np.unique(prob.mesh.elem_nodes[sample])
    assert np.array_equal(part["F1"][:, nodes], full["F1"][:, nodes]) or \
        np.abs(part["F1"][:, nodes] - full["F1"][:, nodes]).max() < 1e-14 * full["F1mag"].max()
    assert np.array_equal(part["FTw"][cl], full["FTw"][cl])


# --------------------------------------------------------------------------- brute force (P11)
@pytest.mark.parametrize("case", ["2d_q2_2x2", "3d_q2_1", "3d_q3_1"])
def test_P11_bruteforce_mpmath(oracle_lib, case):
    """P11: oracle vs a 40-digit dense evaluation of the definition."""
    from tests import mp_bruteforce as MB
    if case == "2d_q2_2x2":
        prob = W.sedov_like(900, 2, (2, 2), (0, 0), (0.5, 0.5), delta=0.1, e_floor=0.3,
                            vmode="uniform", vscale=0.2)
    elif case == "3d_q2_1":
        prob = W.sedov_like(901, 3, (1, 1, 1), (0,) * 3, (0.2, 0.25, 0.3), delta=0.0,
                            e_floor=0.3, vmode="uniform", vscale=0.2)
        rng = np.random.default_rng(1)
        prob.x = prob.x + 0.01 * rng.standard_normal(prob.x.shape)   # curved element
        prob.mesh.x0 = prob.x.copy()
    else:
        prob = W.triple_point(902, (1, 1, 1), hi=(0.5, 0.5, 0.5))
        rng = np.random.default_rng(2)
        prob.x = prob.x + 0.005 * rng.standard_normal(prob.x.shape)
    r = oracle_lib.force(prob)
    b = MB.evaluate(prob)
    F1b = np.array([[float(t) for t in row] for row in b["F1"]])
    assert np.abs(r["F1"] - F1b).max() <= 1e-13 * r["F1mag"].max()
    for K, vals in b["FTw"].items():
        fb = np.array([float(t) for t in vals])
        assert np.abs(r["FTw"][K] - fb).max() <= 1e-13 * r["FTwmag"][K].max()
    assert abs(r["dt"] - float(b["dt"])) <= 1e-14 * float(b["dt"])


# --------------------------------------------------------------------------- ROM (P14)
def test_rom_lift_project_pins(oracle_lib):
    """P14: lifting a unit reduced vector returns that column of Phi exactly (plus
    the offset); projection through P = pinv(Phi_S) recovers the coefficients of a
    field in range(Phi_S), maps 0 to 0 and matches the normal equations."""
    rng = np.random.default_rng(11)
    Phi, _ = np.linalg.qr(rng.standard_normal((500, 40)))
    Y = np.zeros((40, 5))
    for b in range(5):
        Y[7 * b, b] = 1.0
    out = oracle_lib.lift(Phi, np.zeros(500), Y)
    for b in range(5):
        assert np.array_equal(out[:, b], Phi[:, 7 * b])
    os_ = rng.standard_normal((500, 5))
    out = oracle_lib.lift(Phi, os_, np.zeros((40, 5)))
    assert np.array_equal(out, os_)
    rows = np.sort(rng.choice(500, 120, replace=False))
    PhiS = Phi[rows]
    P = np.linalg.pinv(PhiS)
    c = rng.standard_normal((40, 3))
    f = PhiS @ c
    assert np.abs(oracle_lib.project(P, f) - c).max() < 1e-12
    assert np.all(oracle_lib.project(P, np.zeros((120, 3))) == 0)
    g = rng.standard_normal((120, 3))
    ne = np.linalg.solve(PhiS.T @ PhiS, PhiS.T @ g)
    assert np.abs(oracle_lib.project(P, g) - ne).max() < 1e-12

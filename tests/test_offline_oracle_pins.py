"""Pins of the offline-phase oracle (oracle/offline.py) against what the
paper and the mathematics fix, independently of its own formulas:

P26 POD of snapshots with a known SVD (S^T = Q1 diag(s) Q2^T from random orthogonal factors):
    the singular values are s, the energy criterion picks the closed-form k for thresholds on
    either side of each partial sum, and the basis spans Q1's leading columns;
P27 the POD basis is orthonormal and reproduces every snapshot of an exactly rank-r set;
    with eps = 1 its size is the numerical rank r (DESIGN R31);
P28 DEIM on a permuted identity basis returns the permutation (each column's only nonzero);
P29 the DEIM interpolation property: f in span(U) is reproduced exactly from its sampled
    rows, U (P^T U)^-1 P^T f = f, and the indices are distinct;
P30 the first DEIM index is the position of the largest |u_1| entry (Algorithm 1, step 1).
"""
from __future__ import annotations

import numpy as np

from oracle import offline


def _known_svd(N=300, ns=12, seed=0):
    rng = np.random.default_rng(seed)
    Q1, _ = np.linalg.qr(rng.standard_normal((N, ns)))
    Q2, _ = np.linalg.qr(rng.standard_normal((ns, ns)))
    s = np.array([10.0 / 2 ** i for i in range(ns)])
    return (Q1 * s) @ Q2.T, Q1, s   # S^T [N][ns]


def test_P26_pod_known_svd_and_energy_criterion():
    St, Q1, s = _known_svd()
    S = np.ascontiguousarray(St.T)
    Phi, sig = offline.pod(S, eps=1.0)
    np.testing.assert_allclose(sig, s, rtol=1e-12)
    part = np.cumsum(s) / s.sum()
    for k in (1, 3, 6):
        # a threshold just below the k-th partial sum selects k, just above selects k + 1
        assert offline.pod(S, eps=part[k - 1] - 1e-12)[0].shape[1] == k
        assert offline.pod(S, eps=part[k - 1] + 1e-12)[0].shape[1] == k + 1
    Phi, _ = offline.pod(S, eps=part[4] - 1e-12)
    P1 = Q1[:, :5] @ Q1[:, :5].T
    np.testing.assert_allclose(Phi @ Phi.T, P1, atol=1e-12)


def test_P27_pod_orthonormal_and_reproduces_rank_r():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((500, 4))
    S = np.ascontiguousarray((A @ rng.standard_normal((4, 9))).T)   # 9 snapshots of rank 4
    Phi, sig = offline.pod(S, eps=1.0 - 1e-14, max_k=4)
    assert Phi.shape[1] == 4
    np.testing.assert_allclose(Phi.T @ Phi, np.eye(4), atol=1e-13)
    np.testing.assert_allclose(Phi @ (Phi.T @ S.T), S.T, atol=1e-11 * np.abs(S).max())
    assert sig[4:].max() <= 1e-12 * sig[0]


def test_P27b_pod_eps_one_gives_numerical_rank():
    """eps = 1 keeps every numerically nonzero direction (DESIGN R31): on a rank-r snapshot
    set (near-duplicate snapshots included) the basis has exactly r columns, whose span holds
    every snapshot."""
    rng = np.random.default_rng(7)
    for r, ns in ((3, 10), (6, 16)):
        A = rng.standard_normal((700, r))
        S = (A @ rng.standard_normal((r, ns))).T
        S = np.ascontiguousarray(np.concatenate([S, S[:2] * (1 + 1e-15)]))   # near-duplicates
        Phi, sig = offline.pod(S, eps=1.0)
        assert Phi.shape[1] == r
        np.testing.assert_allclose(Phi @ (Phi.T @ S.T), S.T, atol=1e-11 * np.abs(S).max())


def test_P28_deim_permutation_basis():
    rng = np.random.default_rng(2)
    N, m = 40, 7
    perm = rng.permutation(N)[:m]
    U = np.zeros((N, m))
    U[perm, np.arange(m)] = rng.uniform(0.5, 2.0, m)
    np.testing.assert_array_equal(offline.deim(U), perm)


def test_P29_deim_interpolates_span():
    rng = np.random.default_rng(3)
    U, _ = np.linalg.qr(rng.standard_normal((200, 9)))
    p = offline.deim(U)
    assert len(set(p.tolist())) == 9
    f = U @ rng.standard_normal(9)
    rec = U @ np.linalg.solve(U[p], f[p])
    np.testing.assert_allclose(rec, f, atol=1e-12)


def test_P30_deim_first_index():
    rng = np.random.default_rng(4)
    U = rng.standard_normal((100, 5))
    assert offline.deim(U)[0] == int(np.argmax(np.abs(U[:, 0])))


def test_P31_qdeim_scaled_permutation_basis():
    """Rows that are scaled unit vectors: the pivoted QR takes them in decreasing norm order
    (each pivot leaves the other rows' residuals untouched, they are orthogonal)."""
    rng = np.random.default_rng(5)
    N, m = 40, 7
    rows = rng.permutation(N)[:m]
    scale = np.sort(rng.uniform(0.5, 2.0, m))[::-1]
    U = np.zeros((N, m))
    U[rows, rng.permutation(m)] = scale
    np.testing.assert_array_equal(offline.qdeim(U), rows)


def test_P32_qdeim_matches_brute_force_pivoted_gram_schmidt():
    """Brute force on a small case: pivoted Gram-Schmidt on the rows of U written out (the
    textbook definition of QR with column pivoting applied to U^T), and the interpolation
    property of the selected rows."""
    rng = np.random.default_rng(6)
    U, _ = np.linalg.qr(rng.standard_normal((30, 6)))
    R = U.copy()
    piv = []
    for _ in range(6):
        nrm = [float(R[r] @ R[r]) for r in range(30)]
        p = max(range(30), key=lambda r: (nrm[r], -r))
        piv.append(p)
        q = R[p] / np.sqrt(nrm[p])
        for r in range(30):
            R[r] = R[r] - (R[r] @ q) * q
    np.testing.assert_array_equal(offline.qdeim(U), piv)
    f = U @ rng.standard_normal(6)
    np.testing.assert_allclose(U @ np.linalg.solve(U[piv], f[piv]), f, atol=1e-12)


def test_P33_oversampled_with_ns_equal_m_is_deim():
    rng = np.random.default_rng(7)
    U, _ = np.linalg.qr(rng.standard_normal((300, 8)))
    np.testing.assert_array_equal(offline.deim_oversampled(U, 8), offline.deim(U))


def test_P34_oversampled_first_rows_and_gappy_reconstruction():
    """Column 0 adds the rows of largest |u_0| in decreasing order (closed form); with
    n_s > m the sampled rows give an exact gappy (least-squares) reconstruction of anything
    in span(U), and no row is chosen twice."""
    rng = np.random.default_rng(8)
    N, m, n_s = 250, 6, 15
    U, _ = np.linalg.qr(rng.standard_normal((N, m)))
    I = offline.deim_oversampled(U, n_s)
    assert len(I) == n_s and len(set(I.tolist())) == n_s
    n0 = n_s // m + 1                      # column 0 gets the remainder's extra row
    np.testing.assert_array_equal(I[:n0], np.argsort(-np.abs(U[:, 0]), kind="stable")[:n0])
    f = U @ rng.standard_normal(m)
    c = np.linalg.lstsq(U[I], f[I], rcond=None)[0]
    np.testing.assert_allclose(U @ c, f, atol=1e-12)

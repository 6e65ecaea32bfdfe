"""CPU oracle of the ROM offline phase -- TEST INFRASTRUCTURE ONLY (same
import rules as oracle/__init__.py).

PAPER Sec. 4.3 (POD) and 4.5 (DEIM):

* pod(S, eps): the thin SVD of the snapshot matrix (here S holds one snapshot per row, so the
  paper's snapshot matrix is S^T) by a library SVD (a primitive as a step), the leading k left
  singular vectors with k the smallest integer such that sum_{i<=k} sigma_i / sum_i sigma_i
  >= eps (Eq. energy_criteria), each column signed so that the largest-magnitude entry of
  the matching right singular vector is positive (the convention hydro_pod documents).
* deim(U): Algorithm 1 of Chaturantabut-Sorensen as the paper describes it: p_1 = argmax
  |u_1|; for j >= 2, c solves (P^T U_{<j}) c = P^T u_j and p_j = argmax |u_j - U_{<j} c|
  (numpy.argmax: the first maximum, i.e. the lowest row on ties).

* qdeim(U): Q-DEIM (Drmac-Gugercin): the first m column pivots of a QR
  factorisation with column pivoting of U^T, by a library pivoted QR (scipy.linalg.qr,
  pivoting=True -- LAPACK dgeqp3, a primitive as a step).

* deim_oversampled(U, n_s): the greedy that allows over-sampling (DESIGN.md
  R28): basis column j adds floor(n_s/m) (+1 while j < n_s mod m) rows, those outside the
  sample set I with the largest |u_j - U_{<j} c| (c = numpy.linalg.lstsq of U[I,<j] c ~
  U[I,j]), one at a time in decreasing order (ties: the lowest row).

Pinned by tests/test_offline_oracle_pins.py (closed-form low-rank snapshots, the DEIM
interpolation property, permutation bases)."""
from __future__ import annotations

import numpy as np


def pod(S: np.ndarray, eps: float = 0.9999, max_k: int | None = None):
    """(Phi [N][k], sigma [ns]) of the snapshots S [ns][N]."""
    ns = S.shape[0]
    U, sig, Vt = np.linalg.svd(S.T, full_matrices=False)   # S^T = U diag(sig) Vt
    tot = sig.sum()
    k = ns
    run = 0.0
    for i in range(ns):
        run += sig[i]
        if tot > 0 and run / tot >= eps:
            k = i + 1
            break
    if max_k is not None:
        k = min(k, max_k)
    # numerical rank (DESIGN R31): directions with sigma_i^2 <= ns eps_mach sigma_1^2 are
    # rounding noise of the snapshot set (the Gram route the GPU takes cannot resolve them)
    floor = ns * np.finfo(np.float64).eps * sig[0] ** 2 if sig.size else 0.0
    while k > 0 and not sig[k - 1] ** 2 > floor:
        k -= 1
    V = Vt.T
    for c in range(k):
        imax = int(np.argmax(np.abs(V[:, c])))
        if V[imax, c] < 0:
            U[:, c] = -U[:, c]
    return U[:, :k].copy(), sig


def deim(U: np.ndarray) -> np.ndarray:
    """Greedy DEIM indices [m] of the basis U [N][m]."""
    N, m = U.shape
    p = [int(np.argmax(np.abs(U[:, 0])))]
    for j in range(1, m):
        A = U[p, :j]
        c = np.linalg.solve(A, U[p, j])
        r = U[:, j] - U[:, :j] @ c
        p.append(int(np.argmax(np.abs(r))))
    return np.array(p, dtype=np.int64)


def qdeim(U: np.ndarray) -> np.ndarray:
    """Q-DEIM indices [m] of the basis U [N][m]: the first m pivots of U^T P = Q R."""
    import scipy.linalg
    m = U.shape[1]
    _, _, piv = scipy.linalg.qr(U.T, mode="economic", pivoting=True)
    return np.asarray(piv[:m], dtype=np.int64)


def deim_oversampled(U: np.ndarray, n_s: int) -> np.ndarray:
    """Oversampled greedy indices [n_s] of the basis U [N][m], in selection order."""
    N, m = U.shape
    I: list[int] = []
    for j in range(m):
        if j == 0:
            r = U[:, 0]
        else:
            c = np.linalg.lstsq(U[I, :j], U[I, j], rcond=None)[0]
            r = U[:, j] - U[:, :j] @ c
        a = np.abs(r)
        n_add = n_s // m + (1 if j < n_s % m else 0)
        for _ in range(n_add):
            am = a.copy()
            am[I] = -1.0                      # rows already in I are not candidates
            I.append(int(np.argmax(am)))      # the first maximum: the lowest row on ties
    return np.array(I, dtype=np.int64)

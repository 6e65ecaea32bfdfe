"""CPU oracle for the corner-force hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg
and `--impl reference`) may import this package.  The product path
(`paper_2104_11404_b200`) never imports it, and it never imports the product.

Contents:
  tables.py       -- 1D GL / GLL / L2 tables by mpmath (50 digits), rounded once.
  hydro_oracle.c  -- plain C implementation of F.1, F^T.w, dt (see its header for
                     the PAPER.md citations), the ROM lift and projection as naive
                     loops. Built with gcc -O2 -ffp-contract=off (explicit fma()).
  fom.py          -- the full-order RK2-average step: mass matrices by
                     their definition (np.kron tables, scipy.sparse assembly), sparse
                     direct solves, the force via hydro_oracle.c.
  rom.py          -- the hyper-reduced ROM RK2-average online step: naive
                     lifts and projections around the sampled force (NEXT-2).
Parity pins for every function live in tests/test_oracle_pins.py.  Nothing here is
"parity unpinned" except the physical fidelity of readings R3/R5 to Dobrev 2012
(DESIGN.md), which no available source can check.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

from . import tables as _tables

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hydro_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

MAXN, MAXQ, MAXM = 4, 6, 3


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _lib.oracle_lmin3.restype = ctypes.c_double
        _lib.oracle_det.restype = ctypes.c_double
        _lib.oracle_force.restype = ctypes.c_int
    return _lib


class _Tab(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("k", ctypes.c_int), ("q", ctypes.c_int),
                ("xi", ctypes.c_double * MAXQ), ("w", ctypes.c_double * MAXQ),
                ("B", (ctypes.c_double * MAXN) * MAXQ), ("G", (ctypes.c_double * MAXN) * MAXQ),
                ("Bl", (ctypes.c_double * MAXM) * MAXQ)]


def make_tab(dim: int, k: int, q: int) -> _Tab:
    T = _tables.tables(k, q)
    t = _Tab()
    t.dim, t.k, t.q = dim, k, q
    for i in range(q):
        t.xi[i] = T["xi"][i]
        t.w[i] = T["w"][i]
        for a in range(k + 1):
            t.B[i][a] = T["B"][i][a]
            t.G[i][a] = T["G"][i][a]
        for j in range(k):
            t.Bl[i][j] = T["Bl"][i][j]
    assert lib().oracle_sizeof_tab() == ctypes.sizeof(_Tab)
    return t


def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def lmin3(a6) -> float:
    """Contract A.4 smallest eigenvalue of [a00 a11 a22 a01 a02 a12]."""
    arr = (ctypes.c_double * 6)(*[float(x) for x in a6])
    return lib().oracle_lmin3(arr)


def det(dim: int, J) -> float:
    J = np.zeros((3, 3)) + 0.0 if J is None else np.asarray(J, dtype=np.float64)
    M = np.zeros((3, 3))
    M[:J.shape[0], :J.shape[1]] = J
    arr = (ctypes.c_double * 9)(*M.ravel().tolist())
    return lib().oracle_det(dim, arr)


def force(prob, elist: Optional[np.ndarray] = None, mode: int = 0, nthreads: int = 0,
          x=None, v=None, e=None, w=None, want_dtq: bool = False) -> dict:
    """Evaluate F.1 (assembled), F^T.w (element-local), dt on `prob` (a
    workloads.Problem). `elist` restricts the element loop (sorted ids).
    Overrides x/v/e/w replace the problem's state arrays."""
    L = lib()
    m = prob.mesh
    dim = m.dim
    tab = make_tab(dim, m.k, m.nq)
    xs = np.ascontiguousarray(prob.x if x is None else x, dtype=np.float64)
    vs = np.ascontiguousarray(prob.v if v is None else v, dtype=np.float64)
    es = np.ascontiguousarray(prob.e if e is None else e, dtype=np.float64)
    ww = prob.w if w is None else w
    ws = None if ww is None else np.ascontiguousarray(ww, dtype=np.float64)
    x0 = np.ascontiguousarray(m.x0)
    en = np.ascontiguousarray(m.elem_nodes, dtype=np.int32)
    rho0 = np.ascontiguousarray(m.rho0, dtype=np.float64)
    gam = np.ascontiguousarray(prob.gamma, dtype=np.float64)
    el = None if elist is None else np.ascontiguousarray(elist, dtype=np.int32)
    n_list = m.n_elem if el is None else el.size
    nq = m.nq ** dim
    F1 = F1mag = FTw = FTwmag = None
    if mode == 0:
        F1 = np.zeros((dim, m.n_nodes))
        F1mag = np.zeros((dim, m.n_nodes))
        FTw = np.full((m.n_elem, m.ne), np.nan) if el is not None else np.zeros((m.n_elem, m.ne))
        FTwmag = np.zeros((m.n_elem, m.ne))
    dt = ctypes.c_double(0.0)
    bad = ctypes.c_int64(0)
    dtq = np.zeros((n_list, nq)) if want_dtq else None
    rc = L.oracle_force(ctypes.byref(tab), ctypes.c_int64(m.n_elem), ctypes.c_int64(m.n_nodes),
                        _p(en), _p(x0), _p(rho0), _p(xs), _p(vs), _p(es), _p(ws), _p(gam),
                        ctypes.c_int(1 if prob.visc else 0), ctypes.c_double(prob.q1),
                        ctypes.c_double(prob.q2), ctypes.c_double(prob.alpha),
                        ctypes.c_double(prob.alpha_mu), _p(el), ctypes.c_int64(n_list),
                        ctypes.c_int(mode), _p(F1), _p(FTw), _p(F1mag), _p(FTwmag),
                        ctypes.byref(dt), ctypes.byref(bad), _p(dtq), ctypes.c_int(nthreads))
    out = dict(F1=F1, FTw=FTw, F1mag=F1mag, FTwmag=FTwmag, dt=dt.value, first_bad=bad.value,
               status=rc)
    if want_dtq:
        out["dtq"] = dtq
    return out


def lift(Phi: np.ndarray, os_: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """out[r][b] = os[r](or os[r][b]) + sum_k Phi[r][k] Y[k][b] (naive loops)."""
    rows, n = Phi.shape
    B = Y.shape[1]
    out = np.empty((rows, B))
    batched = 1 if os_.ndim == 2 else 0
    lib().oracle_lift(ctypes.c_int64(rows), ctypes.c_int(n), ctypes.c_int(B),
                      _p(np.ascontiguousarray(Phi)), _p(np.ascontiguousarray(os_)),
                      ctypes.c_int(batched), _p(np.ascontiguousarray(Y)), _p(out))
    return out


def project(P: np.ndarray, f: np.ndarray) -> np.ndarray:
    """r[i][b] = sum_s P[i][s] f[s][b] (naive loops)."""
    n, s = P.shape
    B = f.shape[1]
    r = np.empty((n, B))
    lib().oracle_project(ctypes.c_int(n), ctypes.c_int64(s), ctypes.c_int(B),
                         _p(np.ascontiguousarray(P)), _p(np.ascontiguousarray(f)), _p(r))
    return r


def lmin3_stats(reset: bool = True):
    """(Jacobi rotations performed, lmin3 calls) accumulated by oracle.force since the
    last reset -- bench.py uses it to count the contract's data-dependent work."""
    r, c = ctypes.c_int64(0), ctypes.c_int64(0)
    lib().oracle_stats(ctypes.byref(r), ctypes.byref(c), ctypes.c_int(1 if reset else 0))
    return r.value, c.value


def lmin3_fallback_stats(reset: bool = True):
    """(Jacobi rotations performed, lmin3 calls, Jacobi fallbacks) accumulated by oracle.force
    since the last reset (DESIGN A.4 / R30: the closed form falls back to Jacobi near a double
    smallest eigenvalue) -- bench.py's work model."""
    r, c, f = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    lib().oracle_stats2(ctypes.byref(r), ctypes.byref(c), ctypes.byref(f), ctypes.c_int(1 if reset else 0))
    return r.value, c.value, f.value


def tables(k: int, q: int) -> dict:
    return _tables.tables(k, q)

"""Seeded synthetic inputs for the corner-force hot path (BASELINE.json configs C0..C4).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle (`oracle/`): it produces meshes (lattices, element->node tables,
perturbed node positions) and states (x, v, e, gamma, rho0). It holds none of
the method's arithmetic -- no basis functions, no quadrature, no Jacobians, no
equation of state.  Every random number comes from SplitMix64 (Steele, Lea,
Flood 2014) in a vectorised numpy form.

Input recipe:
  * stream seed = ((11404 + cfg) << 8) | tag, tags: 0 positions, 1 velocity
    components, 2 velocity magnitudes, 3 sample elements, 4 mu, 5 Yhat,
    6/7/8 Gaussian matrices for Phi_x/Phi_v/Phi_e.
  * draws run in ascending global node (or element) index, then component.
  * lattices are lexicographic with x fastest; element (i,j,l) owns lattice
    nodes (k*i+a1, k*j+a2, k*l+a3), local index a1 + n*a2 + n*n*a3, n = k+1.
  * L2 (energy) dofs are element-major, local lexicographic j1 fastest, m = k
    per dim, placed (for the Gresho profile only) at Gauss-Legendre points of
    the element, which numpy's leggauss provides independently of both sides.

Problem shapes follow PAPER.md Sec. 6.1: Gresho,
Sedov, Taylor-Green, triple point,
with the domains/sizes of BASELINE.json configs.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

TAG_POS, TAG_VCOMP, TAG_VMAG, TAG_SAMPLE, TAG_MU, TAG_YHAT = 0, 1, 2, 3, 4, 5
TAG_PHI_X, TAG_PHI_V, TAG_PHI_E = 6, 7, 8


def stream_seed(cfg: int, tag: int) -> int:
    return (((11404 + cfg) << 8) | tag) & 0xFFFFFFFFFFFFFFFF


def splitmix64(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start..start+n-1 of the SplitMix64 generator seeded with `seed`."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, n: int, start: int = 0) -> np.ndarray:
    """(z >> 11) * 2^-53 in [0, 1)."""
    return (splitmix64(seed, n, start) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm(seed: int, n: int, a: float, start: int = 0) -> np.ndarray:
    """U[-a, a] = a * (2u - 1)."""
    return a * (2.0 * uniform01(seed, n, start) - 1.0)


def normal(seed: int, n: int) -> np.ndarray:
    """Box-Muller on consecutive uniform pairs, cosine branch only."""
    u = uniform01(seed, 2 * n).reshape(n, 2)
    u1 = np.maximum(u[:, 0], 2.0 ** -60)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u[:, 1])


# ----------------------------------------------------------------------------
# meshes
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Mesh:
    dim: int
    k: int                      # H1 order (Q_k); L2 is Q_{k-1}
    nq: int                     # Gauss-Legendre points per dim
    shape: tuple                # elements per dim (nx, ny[, nz])
    lo: tuple
    hi: tuple
    elem_nodes: np.ndarray      # int32 [E][(k+1)^d]
    x0: np.ndarray              # float64 [d][n_nodes] SoA, initial positions
    rho0: np.ndarray            # float64 [E]

    @property
    def n_elem(self) -> int:
        return int(self.elem_nodes.shape[0])

    @property
    def n_nodes(self) -> int:
        return int(self.x0.shape[1])

    @property
    def nd(self) -> int:        # H1 nodes per element
        return (self.k + 1) ** self.dim

    @property
    def ne(self) -> int:        # L2 dofs per element
        return self.k ** self.dim

    @property
    def lattice(self) -> tuple:
        return tuple(self.k * s + 1 for s in self.shape)

    @property
    def h(self) -> tuple:       # nominal (unperturbed) element widths
        return tuple((b - a) / s for a, b, s in zip(self.lo, self.hi, self.shape))

    @property
    def N_V(self) -> int:       # kinematic dofs
        return self.dim * self.n_nodes

    @property
    def N_E(self) -> int:       # thermodynamic dofs
        return self.ne * self.n_elem


def _gll01(k: int) -> np.ndarray:
    """Gauss-Lobatto points on [0,1] from numpy (geometry of the generated lattice)."""
    if k == 1:
        return np.array([0.0, 1.0])
    inner = np.sort(np.polynomial.legendre.Legendre.basis(k).deriv().roots().real)
    return np.concatenate([[0.0], 0.5 * (inner + 1.0), [1.0]])


def lattice_mesh(dim: int, k: int, nq: int, shape: Sequence[int], lo: Sequence[float],
                 hi: Sequence[float]) -> Mesh:
    shape = tuple(int(s) for s in shape)
    assert len(shape) == dim and dim in (2, 3) and k >= 1
    n = k + 1
    L = [k * s + 1 for s in shape]
    # node coordinates, lexicographic x fastest. Inside every element the k+1
    # nodes per dim sit at the Gauss-Lobatto points (numpy roots of P_k'), so a
    # uniform lattice is an affine (straight-sided) mesh for any k.
    gll = _gll01(k)
    axes = []
    for c in range(dim):
        i = np.arange(L[c])
        el, a = np.minimum(i // k, shape[c] - 1), i - k * np.minimum(i // k, shape[c] - 1)
        hc = (hi[c] - lo[c]) / shape[c]
        ax = lo[c] + hc * (el + gll[a])
        ax[-1] = hi[c]
        axes.append(ax)
    if dim == 2:
        X, Y = np.meshgrid(axes[0], axes[1], indexing="xy")        # [L1][L0]
        x0 = np.stack([X.ravel(), Y.ravel()])
    else:
        Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")  # [L2][L1][L0]
        x0 = np.stack([X.ravel(), Y.ravel(), Z.ravel()])
    x0 = np.ascontiguousarray(x0)
    # element -> node table
    if dim == 2:
        ej, ei = np.meshgrid(np.arange(shape[1]), np.arange(shape[0]), indexing="ij")
        ei, ej = ei.ravel(), ej.ravel()
        a2, a1 = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        a1, a2 = a1.ravel(), a2.ravel()
        en = (k * ei[:, None] + a1[None, :]) + L[0] * (k * ej[:, None] + a2[None, :])
    else:
        el, ej, ei = np.meshgrid(np.arange(shape[2]), np.arange(shape[1]), np.arange(shape[0]),
                                 indexing="ij")
        ei, ej, el = ei.ravel(), ej.ravel(), el.ravel()
        a3, a2, a1 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        a1, a2, a3 = a1.ravel(), a2.ravel(), a3.ravel()
        en = ((k * ei[:, None] + a1[None, :]) + L[0] * (k * ej[:, None] + a2[None, :])
              + L[0] * L[1] * (k * el[:, None] + a3[None, :]))
    en = np.ascontiguousarray(en.astype(np.int32))
    E = int(np.prod(shape))
    return Mesh(dim, k, nq, shape, tuple(lo), tuple(hi), en, x0, np.ones(E))


def node_ijk(mesh: Mesh) -> np.ndarray:
    """Lattice indices [d][n_nodes] of every node."""
    L = mesh.lattice
    idx = np.arange(mesh.n_nodes, dtype=np.int64)
    out = []
    for c in range(mesh.dim):
        out.append(idx % L[c])
        idx = idx // L[c]
    return np.stack(out)


def boundary_nodes(mesh: Mesh) -> np.ndarray:
    ijk = node_ijk(mesh)
    b = np.zeros(mesh.n_nodes, dtype=bool)
    for c, Lc in enumerate(mesh.lattice):
        b |= (ijk[c] == 0) | (ijk[c] == Lc - 1)
    return b


def perturb_interior(mesh: Mesh, frac: float, seed: int) -> None:
    """Every lattice node not on the domain boundary moves, per component, by
    U[-frac*h_c, frac*h_c] (h_c = element width). Draw index =
    node*d + c over ALL nodes; boundary draws are discarded."""
    d = mesh.dim
    du = uniform_pm(seed, mesh.n_nodes * d, 1.0).reshape(mesh.n_nodes, d).T
    interior = ~boundary_nodes(mesh)
    for c in range(d):
        mesh.x0[c, interior] += frac * mesh.h[c] * du[c, interior]


def elem_centroids(mesh: Mesh) -> np.ndarray:
    """Nominal (lattice) element centroids [d][E]."""
    E = mesh.n_elem
    idx = np.arange(E, dtype=np.int64)
    out = []
    for c in range(mesh.dim):
        i = idx % mesh.shape[c]
        idx = idx // mesh.shape[c]
        out.append(mesh.lo[c] + (i + 0.5) * mesh.h[c])
    return np.stack(out)


def l2_dof_points(mesh: Mesh) -> np.ndarray:
    """Physical points [d][E*m^d] of the L2 dofs on the UNPERTURBED lattice
    (Gauss-Legendre nodes, numpy.leggauss), element-major, j1 fastest."""
    m = mesh.k
    g, _ = np.polynomial.legendre.leggauss(m)
    g = 0.5 * (g + 1.0)
    E = mesh.n_elem
    idx = np.arange(E, dtype=np.int64)
    base = []
    for c in range(mesh.dim):
        i = idx % mesh.shape[c]
        idx = idx // mesh.shape[c]
        base.append(mesh.lo[c] + i * mesh.h[c])
    if mesh.dim == 2:
        j2, j1 = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
        loc = [g[j1.ravel()], g[j2.ravel()]]
    else:
        j3, j2, j1 = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
        loc = [g[j1.ravel()], g[j2.ravel()], g[j3.ravel()]]
    pts = [(base[c][:, None] + mesh.h[c] * loc[c][None, :]).ravel() for c in range(mesh.dim)]
    return np.stack(pts)


# ----------------------------------------------------------------------------
# problems
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Problem:
    name: str
    mesh: Mesh
    x: np.ndarray            # [d][n_nodes]
    v: np.ndarray            # [d][n_nodes]
    e: np.ndarray            # [E][m^d]   specific internal energy dofs
    gamma: np.ndarray        # [E]
    visc: bool
    q1: float = 0.5          # BASELINE.json C0: mu = rho h (0.5 cs + 2 h |min(lmin(eps),0)|)
    q2: float = 2.0
    alpha: float = 0.5       # CFL constants
    alpha_mu: float = 2.5
    w: Optional[np.ndarray] = None   # F^T w vector; None => w = v

    @property
    def n_qp(self) -> int:
        return self.mesh.n_elem * self.mesh.nq ** self.mesh.dim


def sedov_like(cfg: int, dim: int, shape, lo, hi, delta: float, e_floor: float,
               vmode: str, vscale: float, k: int = 2, nq: int = 4, mu_scale: float = 1.0,
               name: str = "sedov") -> Problem:
    """Sedov-shaped state: rho0=1, gamma=1.4, energy floor
    everywhere and a spike 0.25*mu/h^d (nominal h) in all dofs of the element
    at the origin, perturbed interior nodes, viscous."""
    mesh = lattice_mesh(dim, k, nq, shape, lo, hi)
    if delta > 0:
        perturb_interior(mesh, delta, stream_seed(cfg, TAG_POS))
    x = mesh.x0.copy()
    n = mesh.n_nodes
    if vmode == "uniform":
        v = uniform_pm(stream_seed(cfg, TAG_VCOMP), n * dim, vscale).reshape(n, dim).T.copy()
    elif vmode == "radial":
        mag = vscale * uniform01(stream_seed(cfg, TAG_VMAG), n)
        r = np.sqrt((x ** 2).sum(axis=0))
        with np.errstate(invalid="ignore", divide="ignore"):
            v = np.where(r > 0, mag * x / np.where(r > 0, r, 1.0), 0.0)
    elif vmode == "zero":
        v = np.zeros_like(x)
    else:
        raise ValueError(vmode)
    vol = float(np.prod(mesh.h))
    e = np.full((mesh.n_elem, mesh.ne), e_floor)
    e[0, :] = 0.25 * mu_scale / vol
    gamma = np.full(mesh.n_elem, 1.4)
    return Problem(name, mesh, x, np.ascontiguousarray(v), e, gamma, visc=True)


def gresho_pressure(r: np.ndarray) -> np.ndarray:
    """PAPER P:2619-2627, middle branch read as 9 - 4 ln 0.2 + 12.5 r^2 - 20 r + 4 ln r
    (the garbled '25/2' fails continuity at r=0.2 and r=0.4)."""
    r = np.asarray(r, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        mid = 9.0 - 4.0 * math.log(0.2) + 12.5 * r * r - 20.0 * r + 4.0 * np.log(np.where(r > 0, r, 1.0))
    return np.where(r < 0.2, 5.0 + 12.5 * r * r, np.where(r < 0.4, mid, 3.0 + 4.0 * math.log(2.0)))


def gresho_vphi(r: np.ndarray) -> np.ndarray:
    """PAPER P:2610-2617."""
    r = np.asarray(r, dtype=np.float64)
    return np.where(r < 0.2, 5.0 * r, np.where(r < 0.4, 2.0 - 5.0 * r, 0.0))


def gresho(cfg: int, shape, k: int = 2, nq: int = 4) -> Problem:
    """Gresho-vortex-shaped state on [0,1]^2 centred at (0.5,0.5) (BASELINE C1;
    SURVEY R8), gamma=5/3, rho=1, no artificial viscosity."""
    mesh = lattice_mesh(2, k, nq, shape, (0.0, 0.0), (1.0, 1.0))
    x = mesh.x0.copy()
    dx, dy = x[0] - 0.5, x[1] - 0.5
    r = np.sqrt(dx * dx + dy * dy)
    vphi = gresho_vphi(r)
    with np.errstate(invalid="ignore", divide="ignore"):
        s = np.where(r > 0, vphi / np.where(r > 0, r, 1.0), 0.0)
    v = np.stack([-dy * s, dx * s])
    gam = 5.0 / 3.0
    pts = l2_dof_points(mesh)
    rp = np.sqrt((pts[0] - 0.5) ** 2 + (pts[1] - 0.5) ** 2)
    e = (gresho_pressure(rp) / ((gam - 1.0) * 1.0)).reshape(mesh.n_elem, mesh.ne)
    return Problem("gresho", mesh, x, np.ascontiguousarray(v), np.ascontiguousarray(e),
                   np.full(mesh.n_elem, gam), visc=False)


def triple_point(cfg: int, shape, lo=(0.0, 0.0, 0.0), hi=(7.0, 3.0, 3.0), k: int = 3,
                 nq: int = 6, vscale: float = 0.05) -> Problem:
    """Triple-point-shaped three-state problem (BASELINE C3).
    Regions by nominal element centroid; e = p/((gamma-1) rho)."""
    mesh = lattice_mesh(3, k, nq, shape, lo, hi)
    cx = elem_centroids(mesh)
    left = cx[0] <= 1.0
    top = cx[1] > 1.5
    rho = np.where(left | ~top, 1.0, 0.125)
    p = np.where(left, 1.0, 0.1)
    gam = np.where(left | top, 1.5, 1.4)
    mesh.rho0 = rho.astype(np.float64)
    e_el = p / ((gam - 1.0) * rho)
    e = np.repeat(e_el[:, None], mesh.ne, axis=1)
    n = mesh.n_nodes
    v = uniform_pm(stream_seed(cfg, TAG_VCOMP), n * 3, vscale).reshape(n, 3).T.copy()
    return Problem("triple_point", mesh, mesh.x0.copy(), v, np.ascontiguousarray(e),
                   gam.astype(np.float64), visc=True)


def taylor_green(cfg: int, shape, k: int = 2, nq: int = 4) -> Problem:
    """Taylor-Green-shaped state on [0,1]^3, gamma=5/3, viscous."""
    mesh = lattice_mesh(3, k, nq, shape, (0.0,) * 3, (1.0,) * 3)
    x = mesh.x0.copy()
    pi = math.pi
    v = np.stack([np.sin(pi * x[0]) * np.cos(pi * x[1]) * np.cos(pi * x[2]),
                  -np.cos(pi * x[0]) * np.sin(pi * x[1]) * np.cos(pi * x[2]),
                  np.zeros(mesh.n_nodes)])
    pts = l2_dof_points(mesh)
    p = 100.0 + ((np.cos(2 * pi * pts[0]) + np.cos(2 * pi * pts[1])) * (np.cos(2 * pi * pts[2]) + 2.0) - 2.0) / 16.0
    gam = 5.0 / 3.0
    e = (p / (gam - 1.0)).reshape(mesh.n_elem, mesh.ne)
    return Problem("taylor_green", mesh, x, np.ascontiguousarray(v), np.ascontiguousarray(e),
                   np.full(mesh.n_elem, gam), visc=True)


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------
def config(name: str) -> Problem:
    """Full-size BASELINE.json configs c0..c3 (c4 is built by `rom_batch`)."""
    name = name.lower()
    if name == "c0":
        return sedov_like(0, 2, (8, 8), (0.0, 0.0), (1.0, 1.0), delta=0.10, e_floor=1e-4,
                          vmode="uniform", vscale=0.1, name="c0_sedov2d")
    if name == "c1":
        p = gresho(1, (256, 256))
        p.name = "c1_gresho2d"
        return p
    if name == "c2":
        return sedov_like(2, 3, (64, 64, 64), (0.0,) * 3, (1.2,) * 3, delta=0.05, e_floor=1e-6,
                          vmode="radial", vscale=0.5, name="c2_sedov3d")
    if name == "c3":
        p = triple_point(3, (112, 48, 48))
        p.name = "c3_triple3d"
        return p
    if name == "tg":
        # not a BASELINE.json config: the Taylor-Green state the north star lists (SURVEY
        # 8(f) NEXT-4), on a C2-sized 64^3 Q2/Q1 mesh of the unit cube
        p = taylor_green(5, (64, 64, 64))
        p.name = "tg_3d"
        return p
    raise ValueError(name)


def small(name: str) -> Problem:
    """Config-shaped problems small enough for the oracle to finish in seconds,
    spanning several CUDA tiles with a ragged tail (odd element counts)."""
    name = name.lower()
    if name == "c0":
        return config("c0")
    if name == "c1":
        p = gresho(101, (23, 17))
        p.name = "c1_small"
        return p
    if name == "c2":
        return sedov_like(102, 3, (7, 5, 3), (0.0,) * 3, (7 * 0.01875, 5 * 0.01875, 3 * 0.01875),
                          delta=0.05, e_floor=1e-6, vmode="radial", vscale=0.5, name="c2_small")
    if name == "c3":
        p = triple_point(103, (9, 5, 3), hi=(2.25, 2.5, 1.5))
        p.name = "c3_small"
        return p
    if name == "tg":
        return taylor_green(104, (5, 4, 3))
    raise ValueError(name)


# ----------------------------------------------------------------------------
# C4: hyper-reduced ROM batch (PAPER Sec. 3.3-3.4)
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class RomBatch:
    base: Problem                 # C2-shaped mesh, x0, gamma, offsets for mu=1
    B: int
    mu: np.ndarray                # [B]
    sample_elems: np.ndarray      # int32 sorted unique S0
    closure_elems: np.ndarray     # int32 sorted: S0 + vertex neighbours
    closure_nodes: np.ndarray     # int64 sorted global node ids touched by the closure
    s0_nodes: np.ndarray          # int64 sorted global node ids of S0 elements
    nx: int
    nv: int
    ne: int
    Phi_x: np.ndarray             # [R_h1][nx]  rows = closure H1 rows (c*n_cl + i)
    Phi_v: np.ndarray             # [R_h1][nv]
    Phi_e: np.ndarray             # [R_l2][ne]  rows = closure L2 rows (elem-major)
    x_os: np.ndarray              # [R_h1]      offset (broadcast over instances)
    v_os: np.ndarray              # [R_h1]
    e_os: np.ndarray              # [R_l2][B]   per-instance offsets (mu-dependent spike)
    Yx: np.ndarray                # [nx][B]
    Yv: np.ndarray                # [nv][B]
    Ye: np.ndarray                # [ne][B]


def vertex_closure(mesh: Mesh, sample: np.ndarray) -> np.ndarray:
    """S0 plus every element sharing at least one H1 node with S0."""
    touched = np.zeros(mesh.n_nodes, dtype=bool)
    touched[mesh.elem_nodes[sample].ravel()] = True
    hit = touched[mesh.elem_nodes].any(axis=1)
    return np.nonzero(hit)[0].astype(np.int32)


def orthonormal(seed: int, rows: int, cols: int) -> np.ndarray:
    """Orthonormal basis of the column space of a seeded U[-1,1] matrix (row-major
    fill), by Cholesky-QR applied twice (CholQR2: orthogonal to ~1e-15 for these
    well-conditioned random matrices, and far faster than Householder at 3.5e6 rows)."""
    q = uniform_pm(seed, rows * cols, 1.0).reshape(rows, cols)
    for _ in range(2):
        r = np.linalg.cholesky(q.T @ q).T            # q^T q = r^T r
        q = q @ np.linalg.inv(r)                      # q r^{-1}
    return np.ascontiguousarray(q)


def rom_batch(base: Problem, cfg: int = 4, B: int = 64, frac: float = 0.02, n_red: int = 40,
              mu_lo: float = 0.7, mu_hi: float = 1.3, n_sample: Optional[int] = None) -> RomBatch:
    mesh = base.mesh
    E = mesh.n_elem
    ns = int(round(frac * E)) if n_sample is None else int(n_sample)
    ns = max(1, min(ns, E))
    # partial Fisher-Yates over element ids
    perm = np.arange(E, dtype=np.int64)
    u = uniform01(stream_seed(cfg, TAG_SAMPLE), ns)
    for i in range(ns):
        j = i + int(u[i] * (E - i))
        perm[i], perm[j] = perm[j], perm[i]
    sample = np.sort(perm[:ns]).astype(np.int32)
    closure = vertex_closure(mesh, sample)
    cl_nodes = np.unique(mesh.elem_nodes[closure].ravel()).astype(np.int64)
    s0_nodes = np.unique(mesh.elem_nodes[sample].ravel()).astype(np.int64)
    mu = mu_lo + (mu_hi - mu_lo) * uniform01(stream_seed(cfg, TAG_MU), B)
    d = mesh.dim
    ncl = cl_nodes.size
    R_h1 = d * ncl
    R_l2 = closure.size * mesh.ne
    Phi_x = orthonormal(stream_seed(cfg, TAG_PHI_X), R_h1, n_red)
    Phi_v = orthonormal(stream_seed(cfg, TAG_PHI_V), R_h1, n_red)
    Phi_e = orthonormal(stream_seed(cfg, TAG_PHI_E), R_l2, n_red)
    x_os = np.ascontiguousarray(mesh.x0[:, cl_nodes].reshape(-1))        # row = c*ncl + i
    v_os = np.zeros(R_h1)
    e_base = base.e[closure].reshape(-1)                                  # floor everywhere + mu=1 spike
    e_floor = float(base.e.min())
    spike_el = np.nonzero(closure == 0)[0]
    e_os = np.repeat(e_base[:, None], B, axis=1)
    if spike_el.size:
        rows = spike_el[0] * mesh.ne + np.arange(mesh.ne)
        e_os[rows, :] = 0.25 * mu[None, :] / float(np.prod(mesh.h))
    # reduced coordinates Yhat: bounded perturbations that keep the
    # lifted mesh untangled and e positive
    yu = uniform_pm(stream_seed(cfg, TAG_YHAT), 3 * n_red * B, 1.0).reshape(3, n_red, B)
    sx = 0.05 * (min(mesh.h) / mesh.k) / np.abs(Phi_x).sum(axis=1).max()
    sv = 0.5 / np.abs(Phi_v).sum(axis=1).max()
    se = 0.5 * e_floor / np.abs(Phi_e).sum(axis=1).max()
    return RomBatch(base, B, mu, sample, closure, cl_nodes, s0_nodes, n_red, n_red, n_red,
                    Phi_x, Phi_v, Phi_e, x_os, v_os, np.ascontiguousarray(e_os),
                    np.ascontiguousarray(sx * yu[0]), np.ascontiguousarray(sv * yu[1]),
                    np.ascontiguousarray(se * yu[2]))


def c4(n_sample: Optional[int] = None, B: int = 64, small_mesh: bool = False) -> RomBatch:
    base = small("c2") if small_mesh else config("c2")
    return rom_batch(base, B=B, n_sample=n_sample)


def sampled_row_maps(batch: RomBatch):
    """Closure-row indices of the sampled rows: H1 rows c*n_cl + pos(S0 node) in the
    order of the library's F1_rows (c*n_s0 + i), and L2 rows l*ne + j of the S0
    elements in the order of FTw_rows (s*ne + j)."""
    mesh = batch.base.mesh
    d, ne = mesh.dim, mesh.ne
    ncl = batch.closure_nodes.size
    pos = np.searchsorted(batch.closure_nodes, batch.s0_nodes)
    h1 = np.concatenate([c * ncl + pos for c in range(d)])
    lpos = np.searchsorted(batch.closure_elems, batch.sample_elems)
    l2 = (lpos[:, None] * ne + np.arange(ne)[None, :]).ravel()
    return h1, l2


def next_window(batch: RomBatch, keep: int = 24, seed: int = 77):
    """A second time window for a ROM batch (same mesh, sample and offsets): each field's
    basis keeps its first `keep` columns and replaces the rest by fresh seeded directions,
    re-orthonormalised (CholQR2), so consecutive windows share a subspace (as bases built
    from overlapping snapshot windows do) but are not equal."""
    import copy
    nb = copy.copy(batch)
    rng = np.random.default_rng(seed)
    for name in ("Phi_x", "Phi_v", "Phi_e"):
        P = getattr(batch, name)
        fresh = rng.uniform(-1.0, 1.0, size=(P.shape[0], P.shape[1] - keep))
        fresh -= P[:, :keep] @ (P[:, :keep].T @ fresh)
        Q = np.concatenate([P[:, :keep], fresh], axis=1)
        for _ in range(2):   # CholQR2
            R = np.linalg.cholesky(Q.T @ Q).T
            Q = np.linalg.solve(R.T, Q.T).T
        setattr(nb, name, np.ascontiguousarray(Q))
    return nb

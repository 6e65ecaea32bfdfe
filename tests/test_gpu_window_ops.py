"""GPU parity of the time-window transition operators (hydro_window_ops; PAPER P:1223-1264,
Eq. ic-tw and the M-oblique Eq. ic2-tw) against oracle/rom.py: the new window's reduced
coordinates T Y + c (applied with the GPU lift kernel, hydro.rom_window_transition) against
the oracle's direct evaluation of the equations, with the oracle's own assembled M_V (sparse)
and M_E (blocks).  Bases are random orthonormal columns over the full FOM rows, offsets
per instance (B = 3).  Tolerance 1e-10 of the largest coordinate: the GPU forms T and c from
split-K products and an LU solve with Mhat, the oracle solves with Mhat once; both are
backward-stable, Mhat is well conditioned for these bases."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from tests import gpu_helpers as H  # noqa: E402
from paper_2104_11404_b200 import hydro  # noqa: E402
from oracle import fom as ofom  # noqa: E402
from oracle import rom as orom  # noqa: E402


def _problem(dim):
    if dim == 2:
        return W.sedov_like(61, 2, (9, 7), (0.0, 0.0), (0.9, 0.7), delta=0.08, e_floor=1e-2,
                            vmode="uniform", vscale=0.1, name="win2")
    return W.sedov_like(62, 3, (4, 3, 3), (0.0, 0.0, 0.0), (0.4, 0.3, 0.3), delta=0.08,
                        e_floor=1e-2, vmode="uniform", vscale=0.1, name="win3")


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("field", [0, 1, 2])
def test_window_ops_match_oracle(dim, field):
    prob = _problem(dim)
    m = prob.mesh
    ctx = H.context(prob)
    f = hydro.Fom(ctx, np.zeros(0, dtype=np.int64))
    rng = np.random.default_rng(100 * dim + field)
    if field == 2:
        N = m.n_elem * m.ne
        Me = ofom.mass_e(m)
        M = lambda a: np.einsum("eij,ejk->eik", Me, a.reshape(m.n_elem, m.ne, -1)).reshape(a.shape)  # noqa: E731
    else:
        N = m.dim * m.n_nodes
        Mv, n = ofom.mass_v(m), m.n_nodes   # scalar block; velocity dofs c * n_nodes + node
        M = lambda a: np.concatenate([Mv @ a[c * n:(c + 1) * n] for c in range(m.dim)])  # noqa: E731
    n_new, n_old, B = 7, 6, 3
    Pn = np.linalg.qr(rng.standard_normal((N, n_new)))[0]
    Po = np.linalg.qr(rng.standard_normal((N, n_old)))[0]
    osn, oso = rng.standard_normal((N, B)), rng.standard_normal((N, B))
    Y = rng.standard_normal((n_old, B))
    T, c = hydro.window_ops(H.dev(Pn), H.dev(Po), H.dev(osn), H.dev(oso),
                            fom=f if field else None, field=field)
    Yg = hydro.rom_window_transition(T, c, H.dev(Y)).cpu().numpy()
    if field == 0:
        Yo = orom.window_transition(Pn, Po, osn, oso, Y)
    else:
        Yo = orom.window_transition_oblique(Pn, Po, osn, oso, Y, M)
    np.testing.assert_allclose(Yg, Yo, atol=1e-10 * np.abs(Yo).max())


def test_window_ops_shared_offset_and_mass_e_apply():
    """Shared offsets ([N], B = 1) and hydro_mass_e_apply against the oracle's M_E blocks."""
    prob = _problem(2)
    m = prob.mesh
    ctx = H.context(prob)
    f = hydro.Fom(ctx, np.zeros(0, dtype=np.int64))
    rng = np.random.default_rng(7)
    N = m.n_elem * m.ne
    x = rng.standard_normal(N)
    Me = ofom.mass_e(m)
    ref = np.einsum("eij,ej->ei", Me, x.reshape(m.n_elem, m.ne)).reshape(-1)
    np.testing.assert_allclose(f.mass_e(H.dev(x)).cpu().numpy(), ref, atol=1e-14 * np.abs(ref).max() * 10)
    Pn = np.linalg.qr(rng.standard_normal((N, 4)))[0]
    osn, oso = rng.standard_normal(N), rng.standard_normal(N)
    T, c = hydro.window_ops(H.dev(Pn), H.dev(Pn), H.dev(osn), H.dev(oso), fom=f, field=2)
    assert tuple(c.shape) == (4, 1)
    Y = rng.standard_normal((4, 1))
    Mf = lambda a: np.einsum("eij,ejk->eik", Me, a.reshape(m.n_elem, m.ne, -1)).reshape(a.shape)  # noqa: E731
    Yo = orom.window_transition_oblique(Pn, Pn, osn, oso, Y, Mf)
    np.testing.assert_allclose((T.cpu().numpy() @ Y + c.cpu().numpy()), Yo, atol=1e-10 * np.abs(Yo).max())
    # same basis, same offsets: the identity map
    T2, c2 = hydro.window_ops(H.dev(Pn), H.dev(Pn), H.dev(osn), H.dev(osn), fom=f, field=2)
    np.testing.assert_allclose(T2.cpu().numpy(), np.eye(4), atol=1e-12)
    assert np.all(c2.cpu().numpy() == 0.0)

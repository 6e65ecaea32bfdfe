"""GPU parity of the Theorem-2 a-posteriori integrands (hydro_rom_indicator; PAPER Eq.
aposteriori-semi) against oracle/rom.aposteriori_integrand
(force oracle + dense linear algebra): random orthonormal state bases, force bases sampled by
greedy DEIM (s = m) or oversampled (s > m), on 2D and 3D Q2 meshes at a perturbed state --
and along a short FOM trajectory as the lifted states of a ROM would be.  Tolerance 1e-9
relative to |f|: the GPU forms the projections from split-K products and host LU/QR solves,
the oracle from numpy's."""
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
from oracle import offline as ooff  # noqa: E402
from oracle import rom as orom  # noqa: E402
import oracle  # noqa: E402


def _problem(dim):
    if dim == 2:
        return W.sedov_like(71, 2, (9, 7), (0.0, 0.0), (0.9, 0.7), delta=0.08, e_floor=1e-2,
                            vmode="uniform", vscale=0.1, name="ind2")
    return W.sedov_like(72, 3, (4, 3, 3), (0.0, 0.0, 0.0), (0.4, 0.3, 0.3), delta=0.08,
                        e_floor=1e-2, vmode="uniform", vscale=0.1, name="ind3")


def _bases(m, rng, oversample):
    NV, NE = m.dim * m.n_nodes, m.n_elem * m.ne
    Pv = np.linalg.qr(rng.standard_normal((NV, 6)))[0]
    Pe = np.linalg.qr(rng.standard_normal((NE, 5)))[0]
    U1 = np.linalg.qr(rng.standard_normal((NV, 8)))[0]
    U2 = np.linalg.qr(rng.standard_normal((NE, 7)))[0]
    if oversample:
        Z1, Z2 = ooff.deim_oversampled(U1, 13), ooff.deim_oversampled(U2, 11)
    else:
        Z1, Z2 = ooff.deim(U1), ooff.deim(U2)
    return Pv, Pe, U1, Z1, U2, Z2


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("oversample", [False, True])
def test_indicator_matches_oracle(dim, oversample):
    prob = _problem(dim)
    m = prob.mesh
    ctx = H.context(prob)
    f = hydro.Fom(ctx, np.zeros(0, dtype=np.int64))
    rng = np.random.default_rng(10 * dim + oversample)
    Pv, Pe, U1, Z1, U2, Z2 = _bases(m, rng, oversample)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    eg = f.indicator(H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma), visc, cfl,
                     H.dev(Pv), H.dev(Pe), H.dev(U1), Z1, H.dev(U2), Z2)
    eo = orom.aposteriori_integrand(prob, prob.x, prob.v, prob.e, Pv, Pe, U1, Z1, U2, Z2)
    out = oracle.force(prob, w=prob.v)
    nf = (np.linalg.norm(out["F1"]), np.linalg.norm(out["FTw"]))
    for k in range(2):
        assert abs(eg[k] - eo[k]) <= 1e-9 * nf[k], (k, eg[k], eo[k])
        assert eo[k] > 1e-3 * nf[k]          # random bases: the integrand is far from zero


def test_indicator_along_a_fom_trajectory():
    """The integrand at the states of three FOM steps (standing in for lifted ROM states),
    summed by the left rectangle rule over the steps like the bound's time integral."""
    prob = _problem(2)
    m = prob.mesh
    rng = np.random.default_rng(5)
    prob.e[:] = 1.0 + 0.5 * rng.random(prob.e.shape)
    from oracle import fom as ofom
    bc = ofom.bc_dofs_box(m)
    prob.v.reshape(-1)[bc] = 0.0
    ctx = H.context(prob)
    f = hydro.Fom(ctx, bc)
    Pv, Pe, U1, Z1, U2, Z2 = _bases(m, rng, False)
    x, v, e, g = H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    dt = 0.2 * oracle.force(prob)["dt"]
    ig = io = 0.0
    for _ in range(3):
        eg = f.indicator(x, v, e, g, visc, cfl, H.dev(Pv), H.dev(Pe), H.dev(U1), Z1, H.dev(U2), Z2)
        xs, vs, es = (t.cpu().numpy().reshape(a.shape) for t, a in ((x, prob.x), (v, prob.v), (e, prob.e)))
        eo = orom.aposteriori_integrand(prob, xs, vs, es, Pv, Pe, U1, Z1, U2, Z2)
        np.testing.assert_allclose(eg, eo, rtol=1e-9)
        ig += dt * (eg[0] + eg[1])
        io += dt * (eo[0] + eo[1])
        f.step(x, v, e, g, visc, cfl, dt, cg_tol=1e-14, cg_max_iter=2000)
    assert abs(ig - io) <= 1e-9 * io

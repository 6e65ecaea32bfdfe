"""Pins of the FOM-step oracle (oracle/fom.py) against what the
paper and the mathematics fix, independently of its own formulas:

P15 total mass: 1^T M_V 1 = 1^T M_E 1 = sum_K rho0_K |K| (exact integral of a constant);
P16 first moments: (x-coordinate field)^T M_V 1 = integral of rho x (closed form on an
    affine, uniform-density box: rho |box| x_centroid);
P17 symmetric positive definite M_V and M_E blocks;
P18 discrete total energy 1/2 v^T M_V v + 1^T M_E e conserved by the RK2-average step
     to rounding, with and without the v.n = 0 boundary condition;
P19 a uniform state at rest stays at rest (F.1 is normal on the box boundary and
    cancels inside; F^T v = 0 at v = 0): v stays 0, e and x unchanged;
P20 a mass-matrix solve reproduces a manufactured solution: M_V^{-1}(M_V u) = u on the
    free dofs.
"""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W

sp = pytest.importorskip("scipy")


def _fom():
    from oracle import fom
    return fom


def _box(dim, k, shape, delta=0.0, cfg=31):
    nq = 4 if k == 2 else 6
    hi = tuple(0.1 * s for s in shape)
    return W.sedov_like(cfg, dim, shape, (0.0,) * dim, hi, delta=delta, e_floor=1e-2,
                        vmode="uniform", vscale=0.1, k=k, nq=nq, name="box")


@pytest.mark.parametrize("dim,k,shape", [(2, 2, (3, 2)), (2, 3, (2, 2)), (3, 2, (2, 2, 2)),
                                         (3, 3, (2, 1, 1))])
def test_P15_total_mass(dim, k, shape):
    fom = _fom()
    prob = _box(dim, k, shape, delta=0.1)          # curved (perturbed) elements
    m = prob.mesh
    vol = np.prod(np.array(m.hi) - np.array(m.lo))
    M = fom.mass_v(m)
    ME = fom.mass_e(m)
    one = np.ones(m.n_nodes)
    assert one @ (M @ one) == pytest.approx(vol, rel=1e-13)        # rho0 = 1
    assert ME.sum() == pytest.approx(vol, rel=1e-13)


@pytest.mark.parametrize("dim,k,shape", [(2, 2, (3, 2)), (3, 2, (2, 2, 1))])
def test_P16_first_moments(dim, k, shape):
    fom = _fom()
    prob = _box(dim, k, shape)                     # affine: unperturbed lattice
    m = prob.mesh
    M = fom.mass_v(m)
    vol = np.prod(np.array(m.hi) - np.array(m.lo))
    one = np.ones(m.n_nodes)
    for c in range(dim):
        cen = 0.5 * (m.lo[c] + m.hi[c])
        assert m.x0[c] @ (M @ one) == pytest.approx(vol * cen, rel=1e-13)


def test_P17_spd():
    fom = _fom()
    m = _box(3, 2, (2, 2, 1), delta=0.1).mesh
    M = fom.mass_v(m).toarray()
    assert np.abs(M - M.T).max() <= 1e-15 * np.abs(M).max()
    assert np.linalg.eigvalsh(M).min() > 0
    ME = fom.mass_e(m)
    assert np.allclose(ME, ME.transpose(0, 2, 1), rtol=0, atol=1e-18)
    assert (np.linalg.eigvalsh(ME).min(axis=1) > 0).all()


@pytest.mark.parametrize("dim,k,shape,use_bc", [(2, 2, (4, 3), True), (2, 2, (4, 3), False),
                                                (3, 2, (2, 2, 2), True)])
def test_P18_energy_conservation(oracle_lib, dim, k, shape, use_bc):
    fom = _fom()
    prob = _box(dim, k, shape, delta=0.08)
    m = prob.mesh
    bc = fom.bc_dofs_box(m) if use_bc else np.zeros(0, dtype=np.int64)
    F = fom.Fom(m, bc)
    v = prob.v.copy()
    v.reshape(-1)[bc] = 0.0
    rng = np.random.default_rng(4)
    prob.e[:] = 1.0 + 0.5 * rng.random(prob.e.shape)   # smooth positive energy (no Sedov spike)
    x, e = prob.x.copy(), prob.e.copy()
    E0 = sum(F.energy(v, e))
    dt = 0.2 * oracle_lib.force(prob)["dt"]
    for _ in range(3):
        x, v, e, dt_est = fom.rk2avg_step(F, prob, x, v, e, dt)
        assert np.isfinite(dt_est)
    kin, inte = F.energy(v, e)
    assert kin > 0
    assert abs(kin + inte - E0) <= 1e-12 * E0


def test_P19_rest_state_stays_at_rest(oracle_lib):
    fom = _fom()
    prob = _box(2, 2, (3, 3))
    m = prob.mesh
    prob.v[:] = 0.0
    prob.e[:] = 0.5
    F = fom.Fom(m, fom.bc_dofs_box(m))
    x1, v1, e1, _ = fom.rk2avg_step(F, prob, prob.x.copy(), prob.v.copy(), prob.e.copy(), 1e-3)
    assert np.abs(v1).max() <= 1e-13
    assert np.array_equal(e1, prob.e)
    assert np.abs(x1 - prob.x).max() <= 1e-16


def test_P20_solve_manufactured():
    fom = _fom()
    m = _box(2, 2, (4, 3), delta=0.1).mesh
    bc = fom.bc_dofs_box(m)
    F = fom.Fom(m, bc)
    rng = np.random.default_rng(2)
    u = rng.standard_normal((2, m.n_nodes))
    u.reshape(-1)[bc] = 0.0
    rhs = np.stack([F.M @ u[c] for c in range(2)])
    got = F.solve_v(rhs)
    assert np.abs(got - u).max() <= 1e-12 * np.abs(u).max()


def test_P23_dt_controller_worked_example():
    """The controller of PAPER P:549-566 (beta1 = 0.85, beta2 = 1.02, gamma = 0.8) on a step
    whose estimate is a constant 1.0, from dt = 2.0 over [0, 3]: the trace worked by hand
    from the algorithm's four steps -- rejections 2.0, 1.7, 1.445, 1.22825, 1.0440125
    (each >= 1.0), then 0.887410625 accepted three times (not <= 0.8, so no growth), then
    the shortened last step 3 - 3 * 0.887410625 = 0.337768125 lands on t = 3 and, being
    <= 0.8 * 1.0, grows the next step to 1.02 * 0.337768125."""
    fom = _fom()
    calls = []

    def step(x, v, e, h):
        calls.append(h)
        return x, v, e, 1.0
    x, v, e, t, h, ns, nr = fom.advance(None, None, 0, 0, 0, 0.0, 3.0, 2.0, step=step)
    assert (ns, nr) == (4, 5)
    assert t == 3.0
    want = [2.0, 1.7, 1.445, 1.22825, 1.0440125, 0.887410625, 0.887410625, 0.887410625]
    assert np.allclose(calls[:8], want, rtol=1e-15, atol=0)
    assert np.isclose(calls[8], 3.0 - 3 * 0.887410625, rtol=1e-13)
    assert np.isclose(h, 1.02 * (3.0 - 3 * 0.887410625), rtol=1e-13)


def test_P23_dt_controller_growth_and_max_steps():
    """Estimate 10 x the step: never rejected; every accepted step is <= 0.8 * estimate, so
    the step grows by beta2 = 1.02 each time (h_n = 1.02^n h_0); max_steps stops the loop."""
    fom = _fom()
    hs = []

    def step(x, v, e, h):
        hs.append(h)
        return x, v, e, 10.0 * h
    *_, t, h, ns, nr = fom.advance(None, None, 0, 0, 0, 0.0, 1e9, 0.5, step=step, max_steps=6)
    assert (ns, nr) == (6, 0)
    assert np.allclose(hs, [0.5 * 1.02 ** i for i in range(6)], rtol=1e-15, atol=0)
    assert np.isclose(t, sum(hs), rtol=1e-15)
    assert np.isclose(h, 0.5 * 1.02 ** 6, rtol=1e-15)

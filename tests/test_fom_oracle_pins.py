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


# ---------------------------------------------------------------------------------------
# P39-P41: the stage structure of the RK2-average step (PAPER Eq. RK2-avg).
# P18 (energy) holds for any half-stage state and P19 for any position update, so these
# pin the half-stage state U^{n+1/2} = (v^{n+1/2}, e^{n+1/2}, x^{n+1/2}) and the final
# position update x^{n+1} = x^n + dt vbar on their own.
# ---------------------------------------------------------------------------------------
class _UnitMass:
    """M_V = M_E = 1 (a one-dof system): the solves are the identity."""

    @staticmethod
    def solve_v(r):
        return r

    @staticmethod
    def solve_e(r):
        return r


def _scalar_force(x, v, e, w=None):
    """A 1x1 'force matrix' F = f(x, v, e) = x + e/2 + v/4, so F.1 = f and F^T w = f w --
    the structure of PAPER Eq. fom, under which 1/2 v^2 + e is conserved."""
    f = x + 0.5 * e + 0.25 * v
    return {"F1": f, "FTw": f * (v if w is None else w), "dt": 1.0, "status": 0}


def _worked_example_ok(step) -> bool:
    """P39, worked by hand from PAPER P:463-508 with M = 1, F = x + e/2 + v/4,
    (x, v, e) = (1, 1/2, 1/4), dt = 1/2:
      F(U^n) = 5/4;  v^{n+1/2} = 1/2 - (1/4)(5/4) = 3/16;
      e^{n+1/2} = 1/4 + (1/4)(5/4)(3/16) = 79/256;  x^{n+1/2} = 1 + (1/4)(3/16) = 67/64;
      F(U^{n+1/2}) = 67/64 + 79/512 + 3/64 = 639/512;  v^{n+1} = 1/2 - (1/2)(639/512) = -127/1024;
      vbar = 385/2048;  e^{n+1} = 1/4 + (1/2)(639/512)(385/2048) = 770303/2097152;
      x^{n+1} = 1 + (1/2)(385/2048) = 4481/4096;  1/2 v^2 + e = 3/8 before and after.
    Every value is a short dyadic fraction, so IEEE arithmetic reproduces it exactly."""
    a = lambda t: np.array([[t]], dtype=np.float64)
    x1, v1, e1, _ = step(_UnitMass, None, a(1.0), a(0.5), a(0.25), 0.5, force=_scalar_force)
    return (x1.item() == 4481 / 4096 and v1.item() == -127 / 1024
            and e1.item() == 770303 / 2097152)


def test_P39_rk2avg_worked_example():
    assert _worked_example_ok(_fom().rk2avg_step)


def _const_accel_ok(step) -> bool:
    """P40: a force constant in time -- F.1 = M_V a and F^T w = G^T w for a fixed G -- makes
    the semi-discrete system Newton's law under constant acceleration, whose
    exact solution is v(t) = v - t a, x(t) = x + t v - t^2/2 a,
    M_E e(t) = M_E e + t G^T v - t^2/2 G^T a.  A second-order scheme with the paper's
    stages reproduces it exactly (up to rounding) in one step; the real mass matrices of a
    curved 2D Q2 mesh with v.n = 0 make the solves non-trivial."""
    fom = _fom()
    prob = _box(2, 2, (3, 2), delta=0.1)
    m = prob.mesh
    bc = fom.bc_dofs_box(m)
    F = fom.Fom(m, bc)
    rng = np.random.default_rng(39)
    a = rng.standard_normal((2, m.n_nodes))
    a.reshape(-1)[bc] = 0.0
    Ma = np.stack([F.M @ a[c] for c in range(2)])
    G = rng.standard_normal((m.n_elem * m.ne, 2 * m.n_nodes))

    def force(x, v, e, w=None):
        ww = v if w is None else w
        return {"F1": Ma, "FTw": (G @ ww.reshape(-1)).reshape(m.n_elem, m.ne), "dt": 1.0,
                "status": 0}
    x = prob.x.copy()
    v = rng.standard_normal((2, m.n_nodes))
    v.reshape(-1)[bc] = 0.0
    e = prob.e.copy()
    t = 0.37
    x1, v1, e1, _ = step(F, prob, x, v, e, t, force=force)
    gv = (G @ v.reshape(-1)).reshape(m.n_elem, m.ne)
    ga = (G @ a.reshape(-1)).reshape(m.n_elem, m.ne)
    e_want = e + F.solve_e(t * gv - 0.5 * t * t * ga)
    ok = np.abs(v1 - (v - t * a)).max() <= 1e-12 * np.abs(v).max()
    ok &= np.abs(x1 - (x + t * v - 0.5 * t * t * a)).max() <= 1e-13 * np.abs(x).max()
    ok &= np.abs(e1 - e_want).max() <= 1e-12 * np.abs(e_want).max()
    return bool(ok)


def test_P40_rk2avg_constant_acceleration():
    assert _const_accel_ok(_fom().rk2avg_step)


def _order_ratio(step):
    """P41: temporal self-convergence of the step with the real corner force on a smooth
    inviscid state (Gresho-shaped, 6x5 Q2/Q1, v.n = 0): integrate over T = 2 dt_est with
    n = 8, 16, 32 steps; for a second-order scheme ||y_8 - y_16|| / ||y_16 - y_32|| -> 4
    (measured 4.4 here), a first-order one gives ~2."""
    import oracle
    fom = _fom()
    prob = W.gresho(101, (6, 5))
    m = prob.mesh
    bc = fom.bc_dofs_box(m)
    F = fom.Fom(m, bc)
    v0 = prob.v.copy()
    v0.reshape(-1)[bc] = 0.0
    T = 2.0 * oracle.force(prob)["dt"]
    ys = []
    for n in (8, 16, 32):
        x, v, e = prob.x.copy(), v0.copy(), prob.e.copy()
        for _ in range(n):
            x, v, e, _ = step(F, prob, x, v, e, T / n)
        ys.append(np.concatenate([x.ravel(), v.ravel(), e.ravel()]))
    return np.abs(ys[0] - ys[1]).max() / np.abs(ys[1] - ys[2]).max()


def test_P41_rk2avg_second_order(oracle_lib):
    assert 3.0 < _order_ratio(_fom().rk2avg_step) < 5.5


# Seeded mutations of the oracle's own source: each must turn at least one of P39-P41 red.
_MUTATIONS = {
    "x1 uses v^{n+1}": ("x1 = x + dt * vbar", "x1 = x + dt * v1"),
    "x1 uses v^n": ("x1 = x + dt * vbar", "x1 = x + dt * v"),
    "x_h uses v^n": ("x_h = x + 0.5 * dt * v_h", "x_h = x + 0.5 * dt * v"),
    "x_h full step": ("x_h = x + 0.5 * dt * v_h", "x_h = x + dt * v_h"),
    "stage-2 force at v^n": ("s2 = force(x_h, v_h, e_h)", "s2 = force(x_h, v, e_h)"),
    "stage-2 force at e^n": ("s2 = force(x_h, v_h, e_h)", "s2 = force(x_h, v_h, e)"),
    "stage-2 force at x^n": ("s2 = force(x_h, v_h, e_h)", "s2 = force(x, v_h, e_h)"),
    "stage-1 F^T v^n": ("s1w = force(x, v, e, v_h)", "s1w = force(x, v, e, v)"),
    "stage-2 F^T v^{n+1}": ("s2w = force(x_h, v_h, e_h, vbar)", "s2w = force(x_h, v_h, e_h, v1)"),
    "stage-2 F^T v^{n+1/2}": ("s2w = force(x_h, v_h, e_h, vbar)", "s2w = force(x_h, v_h, e_h, v_h)"),
    "e_h full step": ("e_h = e + 0.5 * dt * fom", "e_h = e + dt * fom"),
}


@pytest.mark.parametrize("name", sorted(_MUTATIONS))
def test_P39_P41_catch_mutations(oracle_lib, name):
    import inspect
    fom = _fom()
    src = inspect.getsource(fom.rk2avg_step)
    old, new = _MUTATIONS[name]
    assert old in src, f"mutation site not found: {old!r}"
    ns = dict(vars(fom))
    exec(src.replace(old, new), ns)
    mutant = ns["rk2avg_step"]
    caught = (not _worked_example_ok(mutant)) or (not _const_accel_ok(mutant))
    if not caught:
        r = _order_ratio(mutant)
        caught = not (3.0 < r < 5.5)
    assert caught, name

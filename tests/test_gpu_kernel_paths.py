"""GPU parity of every kernel path against the oracle (DESIGN "Kernels"):

* 2D Q2: the one-thread-per-element kernel (force2d), the point-per-thread kernel
  (force_kernel) and the point-per-lane kernel (force2d_pl, q1 per warp) -- forced with
  hydro_set_2d_kernel -- on C0/C1-shaped meshes, w != v,
  dt_estimate, and a batched sample plan (hydro_force_sampled with B > 1);
* degenerate and ragged meshes: one element (every dim/order), and element counts just
  below / at / above the CTA multiples;
* inviscid 3D (no config uses it, the API allows it).

Bars: F.1 within 1e-11, F^T.w within 1e-12 of max(|ref|, M), dt bit-exact
(BASELINE north_star; DESIGN "Tolerances")."""
from __future__ import annotations

import os

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from tests import gpu_helpers as H  # noqa: E402
from paper_2104_11404_b200 import hydro  # noqa: E402


@pytest.fixture(params=["element", "point", "lane"])
def kernel2d(request, set_kernel_2d):
    set_kernel_2d(request.param)
    return request.param


def check(prob, oracle_lib, w=None, ctx=None, what=""):
    if w is not None:
        prob.w = w
    ref = oracle_lib.force(prob)
    got = H.run_full(prob, ctx=ctx, w=w)
    assert got["status"] == 0 and ref["status"] == 0, (got["status"], ref["status"])
    H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, f"{what} F1")
    H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, f"{what} FTw")
    assert H.dt_bitwise(got["dt"], ref["dt"]), (what, got["dt"], ref["dt"])
    return got


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_2d_paths_match_oracle(oracle_lib, kernel2d, name):
    check(W.small(name), oracle_lib, what=f"{name}/{kernel2d}")


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_2d_paths_w_distinct(oracle_lib, kernel2d, name):
    prob = W.small(name)
    rng = np.random.default_rng(5)
    w = np.ascontiguousarray(prob.v + 0.03 * rng.standard_normal(prob.v.shape))
    check(prob, oracle_lib, w=w, what=f"{name}/{kernel2d} w")


def test_2d_paths_bitwise_identical(set_kernel_2d):
    """Both 2D kernels evaluate the same contract and the same backward FMA order."""
    prob = W.small("c0")
    set_kernel_2d("element")
    a = H.run_full(prob)
    set_kernel_2d("point")
    b = H.run_full(prob)
    assert np.array_equal(a["F1"], b["F1"]) and np.array_equal(a["FTw"], b["FTw"])
    assert H.dt_bitwise(a["dt"], b["dt"])


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_2d_dt_estimate(kernel2d, name):
    prob = W.small(name)
    got = H.run_full(prob)
    dt = got["ctx"].dt_estimate(H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma),
                                hydro.Visc(prob.q1, prob.q2, prob.visc),
                                hydro.Cfl(prob.alpha, prob.alpha_mu))
    assert H.dt_bitwise(float(dt.item()), got["dt"])


def test_2d_batched_sampled_matches_oracle(oracle_lib, kernel2d):
    """hydro_force_sampled on a 2D mesh with B = 3 instances (the 2D kernels' batched
    variants): every instance's sampled rows against the oracle on the closure."""
    from tests.test_gpu_rom import gpu_step, oracle_instance
    base = W.small("c0")
    batch = W.rom_batch(base, B=3, n_sample=5, n_red=8)
    g = gpu_step(batch)
    assert g["status"][0] == 0
    for b in range(batch.B):
        F1, F1m, FT, FTm, dt = oracle_instance(oracle_lib, batch, g["xS"], g["vS"], g["eS"], b)
        H.assert_close(g["F1"][:, b], F1, F1m, H.TOL_LOCAL, f"F1_rows b={b}")
        H.assert_close(g["FT"][:, b], FT, FTm, H.TOL_LOCAL, f"FTw_rows b={b}")
        assert H.dt_bitwise(g["dt"][b], dt)


@pytest.mark.parametrize("dim,k", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_single_element(oracle_lib, set_kernel_2d, dim, k):
    """The degenerate mesh of one element (every node on the boundary)."""
    set_kernel_2d("element")
    nq = 4 if k == 2 else 6
    prob = W.sedov_like(7, dim, (1,) * dim, (0.0,) * dim, (1.0,) * dim, delta=0.0, e_floor=1e-3,
                        vmode="uniform", vscale=0.1, k=k, nq=nq, name="one")
    check(prob, oracle_lib, what=f"one element d{dim}k{k}")


@pytest.mark.parametrize("kind", ["element", "lane"])
@pytest.mark.parametrize("shape", [(1,), (7,), (9,), (63,), (64,), (65,), (127,), (129,)])
def test_2d_ragged_counts(oracle_lib, set_kernel_2d, shape, kind):
    """Element counts around the 64-thread CTA of the element kernel and the 8-element CTA
    of the point-per-lane kernel."""
    set_kernel_2d(kind)
    prob = W.sedov_like(8, 2, (shape[0], 1), (0.0, 0.0), (shape[0] / 8.0, 0.125), delta=0.1,
                        e_floor=1e-4, vmode="uniform", vscale=0.1, name="ragged2d")
    check(prob, oracle_lib, what=f"2D {shape}")


@pytest.mark.parametrize("shape", [(5, 1, 1), (13, 11, 11)])
def test_3d_ragged_counts(oracle_lib, shape):
    """Small 3D element counts (fewer elements than SMs; and a 13x11x11 mesh)."""
    n = shape
    prob = W.sedov_like(9, 3, n, (0.0,) * 3, tuple(0.01875 * s for s in n), delta=0.05,
                        e_floor=1e-6, vmode="radial", vscale=0.5, name="ragged3d")
    check(prob, oracle_lib, what=f"3D {shape}")


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_3d_paths_match_oracle(oracle_lib, name):
    check(W.small(name), oracle_lib, what=name)


def test_3d_batched_sampled_matches_oracle(oracle_lib):
    """hydro_force_sampled on a C2-shaped mesh with B = 3 instances."""
    from tests.test_gpu_rom import gpu_step, oracle_instance
    base = W.small("c2")
    batch = W.rom_batch(base, B=3, n_sample=4, n_red=8)
    g = gpu_step(batch)
    assert g["status"][0] == 0
    for b in range(batch.B):
        F1, F1m, FT, FTm, dt = oracle_instance(oracle_lib, batch, g["xS"], g["vS"], g["eS"], b)
        H.assert_close(g["F1"][:, b], F1, F1m, H.TOL_LOCAL, f"F1_rows b={b}")
        H.assert_close(g["FT"][:, b], FT, FTm, H.TOL_LOCAL, f"FTw_rows b={b}")
        assert H.dt_bitwise(g["dt"][b], dt)


def test_3d_inviscid(oracle_lib):
    prob = W.small("c2")
    prob.visc = False
    check(prob, oracle_lib, what="3D inviscid")

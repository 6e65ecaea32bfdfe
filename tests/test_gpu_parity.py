"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Bars (BASELINE north_star; DESIGN "Tolerances"): assembled F.1 within
1e-11 and element-local F^T.w within 1e-12 of max(|ref|, M) per entry (M = the
oracle's sum of |terms|), dt bit-exact."""
from __future__ import annotations

import math

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from tests import gpu_helpers as H  # noqa: E402


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "tg"])
def test_small_configs_match_oracle(oracle_lib, name):
    prob = W.small(name)
    ref = oracle_lib.force(prob)
    got = H.run_full(prob)
    assert got["status"] == 0 and ref["status"] == 0
    H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, f"{name} F1")
    H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, f"{name} FTw")
    assert H.dt_bitwise(got["dt"], ref["dt"]), (got["dt"], ref["dt"])


def test_w_distinct_from_v(oracle_lib):
    prob = W.small("c2")
    rng = np.random.default_rng(3)
    prob.w = np.ascontiguousarray(prob.v + 0.05 * rng.standard_normal(prob.v.shape))
    ref = oracle_lib.force(prob)
    got = H.run_full(prob, w=prob.w)
    H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, "F1 (w)")
    H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, "FTw (w)")
    assert H.dt_bitwise(got["dt"], ref["dt"])


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_dt_estimate_equals_force_dt(name):
    prob = W.small(name)
    got = H.run_full(prob)
    ctx = got["ctx"]
    dt = ctx.dt_estimate(H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma),
                         H.hydro.Visc(prob.q1, prob.q2, prob.visc), H.hydro.Cfl(prob.alpha, prob.alpha_mu))
    assert H.dt_bitwise(float(dt.item()), got["dt"])


def test_deterministic_bitwise():
    prob = W.small("c2")
    a = H.run_full(prob)
    b = H.run_full(prob, ctx=a["ctx"])
    assert np.array_equal(a["F1"], b["F1"]) and np.array_equal(a["FTw"], b["FTw"])
    assert H.dt_bitwise(a["dt"], b["dt"])


def test_power_of_two_scaling_on_gpu():
    """P6 on the CUDA path: x, x0 -> 2x, 2x0 scales F by 2^(d-1) and dt by 2, bitwise."""
    for name in ("c0", "c2"):
        prob = W.small(name)
        r1 = H.run_full(prob)
        prob.mesh.x0 = prob.mesh.x0 * 2.0
        prob.x = prob.x * 2.0
        r2 = H.run_full(prob)
        d = prob.mesh.dim
        assert np.array_equal(r2["F1"], r1["F1"] * 2.0 ** (d - 1))
        assert np.array_equal(r2["FTw"], r1["FTw"] * 2.0 ** (d - 1))
        assert r2["dt"] == 2 * r1["dt"]


def test_energy_identity_on_gpu():
    prob = W.small("c3")
    r = H.run_full(prob)
    lhs, rhs = (prob.v * r["F1"]).sum(), r["FTw"].sum()
    assert abs(lhs - rhs) <= 1e-12 * (np.abs(prob.v * r["F1"]).sum() + np.abs(r["FTw"]).sum())


def test_tangled_and_nan_status(oracle_lib):
    prob = W.small("c2")
    m = prob.mesh
    for K in (40, 7):
        prob.x[0, m.elem_nodes[K][13]] += 5 * m.h[0]
    got = H.run_full(prob)
    ref = oracle_lib.force(prob, mode=1)
    assert got["status"] == H.hydro.HYDRO_ERR_TANGLED and got["first_bad"] == ref["first_bad"] == 7
    prob = W.small("c2")
    prob.e[3, 2] = np.nan
    got = H.run_full(prob)
    assert got["status"] == H.hydro.HYDRO_ERR_NONFINITE and math.isnan(got["dt"])
    # the sticky status clears; a clean call afterwards reports OK
    got = H.run_full(W.small("c2"), ctx=got["ctx"])
    assert got["status"] == 0 and math.isfinite(got["dt"])


@pytest.mark.parametrize("kind", ["auto", "element", "lane"])
@pytest.mark.parametrize("name", ["c0", "c1"])
def test_full_size_2d_configs(oracle_lib, set_kernel_2d, name, kind):
    """C0 and C1 at their BASELINE.json sizes, every output compared; the size-based kernel
    choice (what the bench times) and each 2D Q2 kernel forced."""
    set_kernel_2d(kind)
    prob = W.config(name)
    ref = oracle_lib.force(prob)
    got = H.run_full(prob)
    H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, f"{name} F1")
    H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, f"{name} FTw")
    assert H.dt_bitwise(got["dt"], ref["dt"])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_size_3d_sampled_outputs(oracle_lib, name):
    """C2 / C3 at full size in the bench's launch configuration: F.1 at 300 sampled
    nodes and F^T.v of 300 sampled elements (oracle on those elements' closures), and
    dt over the whole mesh (oracle dt-only pass), bit-exact."""
    prob = W.config(name)
    got = H.run_full(prob)
    m = prob.mesh
    rng = np.random.default_rng(42)
    nodes = np.unique(rng.choice(m.n_nodes, 300, replace=False))
    mark = np.zeros(m.n_nodes, bool)
    mark[nodes] = True
    elems = np.nonzero(mark[m.elem_nodes].any(axis=1))[0].astype(np.int32)
    sel_e = np.sort(rng.choice(m.n_elem, 300, replace=False)).astype(np.int32)
    elist = np.union1d(elems, sel_e).astype(np.int32)
    ref = oracle_lib.force(prob, elist=elist)
    H.assert_close(got["F1"][:, nodes], ref["F1"][:, nodes], ref["F1mag"][:, nodes],
                   H.TOL_ASSEMBLED, f"{name} F1 sampled")
    H.assert_close(got["FTw"][sel_e], ref["FTw"][sel_e], ref["FTwmag"][sel_e], H.TOL_LOCAL,
                   f"{name} FTw sampled")
    dref = oracle_lib.force(prob, mode=1)
    assert H.dt_bitwise(got["dt"], dref["dt"]), (got["dt"], dref["dt"])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3", "tg"])
def test_full_size_every_output(oracle_lib, name):
    """C3 (3D Q3/Q2, 258 048 elements, the bench's launch configuration with the Q3 layouts and
    task orders) and the Taylor-Green 64^3 workload: every assembled F.1 entry and every F^T.v
    entry against the oracle's full-mesh evaluation, dt bit-exact."""
    prob = W.config(name)
    got = H.run_full(prob)
    ref = oracle_lib.force(prob)
    assert got["status"] == 0 and ref["status"] == 0
    H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, f"{name} F1 (all nodes)")
    H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, f"{name} FTw (all elements)")
    assert H.dt_bitwise(got["dt"], ref["dt"]), (got["dt"], ref["dt"])


@pytest.mark.slow
def test_full_size_c2_every_output(oracle_lib):
    """C2 at its BASELINE.json size in the bench's launch configuration: every assembled F.1
    entry (all 2,146,689 nodes x 3) and every F^T.v entry against the oracle's full-mesh
    evaluation, dt bit-exact."""
    prob = W.config("c2")
    got = H.run_full(prob)
    ref = oracle_lib.force(prob)
    assert got["status"] == 0 and ref["status"] == 0
    H.assert_close(got["F1"], ref["F1"], ref["F1mag"], H.TOL_ASSEMBLED, "c2 F1 (all nodes)")
    H.assert_close(got["FTw"], ref["FTw"], ref["FTwmag"], H.TOL_LOCAL, "c2 FTw (all elements)")
    assert H.dt_bitwise(got["dt"], ref["dt"]), (got["dt"], ref["dt"])

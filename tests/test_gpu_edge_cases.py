"""GPU edge cases of the boundary calls: empty and ragged extents, every lift kernel
path, the empty projection, an empty sample set, and the Q-DEIM cancellation path.

References are the operations' definitions (PAPER P:864-871 for the lift X = x_os + Phi Y,
P:778-799 for the projection r = P f) in extended-precision numpy, or the oracle (`oracle/`);
bars as in test_gpu_rom.py (1e-14 / 1e-13 of the magnitude |terms|)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import workloads as W  # noqa: E402
from oracle import offline as ooff  # noqa: E402
from paper_2104_11404_b200 import hydro  # noqa: E402
from tests import gpu_helpers as H  # noqa: E402


@pytest.mark.parametrize("rows,n,B,batched_os", [
    (1, 1, 1, False), (127, 3, 7, False), (129, 8, 2, True), (1000, 16, 64, False),
    (513, 33, 64, True), (300, 40, 65, False), (257, 64, 64, True), (100, 64, 130, False),
    (64, 65, 4, False), (77, 100, 9, True), (300, 224, 10, False)])
def test_lift_kernel_paths(rows, n, B, batched_os):
    """hydro_rom_lift on each path: the DMMA kernel (n <= 64, even B, shared or per-instance
    offsets; n = 1..64 covers every k-step count, B > 64 several column blocks), the FMA
    fallback (odd B, n > 64); ragged row counts around the 128-row tiles."""
    rng = np.random.default_rng(rows * 31 + n * 7 + B)
    Phi = rng.standard_normal((rows, n))
    Y = rng.standard_normal((n, B))
    os_ = rng.standard_normal((rows, B)) if batched_os else rng.standard_normal(rows)
    got = hydro.rom_lift(H.dev(Phi), H.dev(os_), H.dev(Y)).cpu().numpy()
    os2 = os_ if batched_os else os_[:, None]
    ref = (os2.astype(np.longdouble) + Phi.astype(np.longdouble) @ Y.astype(np.longdouble)).astype(np.float64)
    mag = np.abs(os2) + np.abs(Phi) @ np.abs(Y)
    H.assert_close(got, ref, mag, 1e-14, f"lift rows={rows} n={n} B={B}")


def test_lift_too_many_basis_columns_is_an_argument_error():
    """n beyond the FMA kernel's shared-memory staging (n > 224) is rejected, not launched."""
    Phi = torch.zeros((16, 256), dtype=torch.float64, device="cuda")
    os_ = torch.zeros(16, dtype=torch.float64, device="cuda")
    Y = torch.zeros((256, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(hydro.HydroError):
        hydro.rom_lift(Phi, os_, Y)


def test_lift_zero_rows_is_a_noop():
    Phi = torch.empty((0, 8), dtype=torch.float64, device="cuda")
    os_ = torch.empty((0,), dtype=torch.float64, device="cuda")
    Y = torch.ones((8, 4), dtype=torch.float64, device="cuda")
    out = hydro.rom_lift(Phi, os_, Y)
    torch.cuda.synchronize()
    assert out.shape == (0, 4)


@pytest.mark.parametrize("n,B", [(8, 4), (40, 64), (64, 7)])
def test_project_zero_rows_is_zero(n, B):
    """An empty sample (s = 0 rows): the projection's sum is empty, r = 0 exactly."""
    P = torch.empty((n, 0), dtype=torch.float64, device="cuda")
    f = torch.empty((0, B), dtype=torch.float64, device="cuda")
    r = hydro.rom_project(P, f).cpu().numpy()
    assert r.shape == (n, B) and np.array_equal(r, np.zeros((n, B)))


def test_sample_plan_rejects_an_empty_sample():
    prob = W.small("c2")
    ctx = H.context(prob)
    with pytest.raises(hydro.HydroError):
        hydro.SamplePlan(ctx, np.zeros(0, dtype=np.int32), 2)


def test_qdeim_cancellation_rows_match_lapack():
    """Q-DEIM where downdated row norms cancel: rows that are scaled copies of other rows lose
    their whole residual once their partner is pivoted (the kernel recomputes such norms by
    MGS, as LAPACK's dgeqp3 recomputes its column norms); indices equal to the oracle's
    (scipy / LAPACK pivoted QR of U^T)."""
    rng = np.random.default_rng(77)
    N, m = 20_000, 24
    U, _ = np.linalg.qr(rng.standard_normal((N, m)))
    src = rng.choice(N, 400, replace=False)
    dst = rng.choice(np.setdiff1d(np.arange(N), src), 400, replace=False)
    U[dst] = U[src] * rng.uniform(0.5, 0.99, size=(400, 1))   # never larger than the partner
    U = np.ascontiguousarray(U)
    got = hydro.qdeim(H.dev(U))
    ref = ooff.qdeim(U)
    np.testing.assert_array_equal(got, ref)
    assert len(set(got.tolist())) == m


def test_qdeim_wide_basis_fallback_matches_lapack():
    """m > 64 columns: the residual-rewriting Q-DEIM path (the downdating kernel keeps m <= 64)."""
    rng = np.random.default_rng(70)
    U, _ = np.linalg.qr(rng.standard_normal((3000, 70)))
    U = np.ascontiguousarray(U)
    np.testing.assert_array_equal(hydro.qdeim(H.dev(U)), ooff.qdeim(U))


def test_pod_many_snapshots_fallback_matches_oracle():
    """ns > 64 snapshots: the tiled FMA Gram / basis kernels (the tensor-pipe path takes
    ns <= 64); singular values and the well-separated basis columns against the oracle's SVD,
    orthonormal to 1e-12 after CholQR."""
    rng = np.random.default_rng(80)
    N, ns = 30_001, 80
    Q1, _ = np.linalg.qr(rng.standard_normal((N, ns)))
    Q2, _ = np.linalg.qr(rng.standard_normal((ns, ns)))
    sv = np.array([2.0 / 1.25 ** i for i in range(ns)])
    S = np.ascontiguousarray(((Q1 * sv) @ Q2.T).T)
    Phi_g, sg = hydro.pod(H.dev(S), eps=0.999)
    Phi_o, so = ooff.pod(S, eps=0.999)
    assert Phi_g.shape == Phi_o.shape
    tol = 1e-13 * so[0] ** 2 / np.maximum(so, 1e-300) + 1e-12 * so
    assert np.all(np.abs(sg - so) <= tol)
    P = Phi_g.cpu().numpy()
    k = P.shape[1]
    assert np.abs(P.T @ P - np.eye(k)).max() <= 1e-12
    good = so[:k] >= 1e-3 * so[0]
    Pg, Po = P[:, good], Phi_o[:, good]
    assert np.abs(Pg - Po).max() <= 1e-8

"""GPU parity of the ROM offline phase against
oracle/offline.py: POD by the method of snapshots (hydro_pod) against a library SVD, greedy
DEIM (hydro_deim) index for index, and the pipeline FOM snapshots (incl. the half stages,
P:921-943) -> POD velocity basis -> SNS force basis M_V Phi_v -> DEIM indices.
Tolerances: the Gram route squares the condition number, so a singular value sigma_i is
compared to 1e-13 sigma_1^2 / sigma_i + 1e-12 sigma_i and basis columns only where sigma_i is
well separated; DEIM indices exactly."""
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
from oracle import fom as ofom  # noqa: E402


def _sig_close(sg, so):
    tol = 1e-13 * so[0] ** 2 / np.maximum(so, 1e-300) + 1e-12 * so
    assert np.all(np.abs(sg - so) <= tol), np.max(np.abs(sg - so) / tol)


def test_pod_known_svd_matches_oracle():
    rng = np.random.default_rng(10)
    N, ns = 100_003, 24
    Q1, _ = np.linalg.qr(rng.standard_normal((N, ns)))
    Q2, _ = np.linalg.qr(rng.standard_normal((ns, ns)))
    s = np.array([3.0 / 1.6 ** i for i in range(ns)])
    S = np.ascontiguousarray(((Q1 * s) @ Q2.T).T)
    for eps in (0.9, 0.9999):
        Phi_g, sg = hydro.pod(H.dev(S), eps=eps)
        Phi_o, so = ooff.pod(S, eps=eps)
        assert Phi_g.shape == Phi_o.shape
        _sig_close(sg, so)
        Pg = Phi_g.cpu().numpy()
        k = Pg.shape[1]
        np.testing.assert_allclose(Pg.T @ Pg, np.eye(k), atol=1e-12)
        good = so[:k] >= 1e-3 * so[0]
        np.testing.assert_allclose(Pg[:, good], Phi_o[:, good], atol=1e-8)


@pytest.mark.parametrize("N,m", [(50_000, 20), (7, 7), (1_000, 1)])
def test_deim_matches_oracle(N, m):
    rng = np.random.default_rng(11 + m)
    U, _ = np.linalg.qr(rng.standard_normal((N, m)))
    U = np.ascontiguousarray(U)
    np.testing.assert_array_equal(hydro.deim(H.dev(U)), ooff.deim(U))


@pytest.mark.parametrize("N,m", [(50_000, 20), (9, 5), (1_000, 1), (200_000, 40)])
def test_qdeim_matches_oracle(N, m):
    rng = np.random.default_rng(21 + m)
    U, _ = np.linalg.qr(rng.standard_normal((N, m)))
    U = np.ascontiguousarray(U)
    np.testing.assert_array_equal(hydro.qdeim(H.dev(U)), ooff.qdeim(U))


@pytest.mark.parametrize("N,m,n_s", [(50_000, 20, 40), (50_000, 20, 53), (1_000, 4, 4), (12, 3, 12)])
def test_deim_oversampled_matches_oracle(N, m, n_s):
    rng = np.random.default_rng(31 + n_s)
    U, _ = np.linalg.qr(rng.standard_normal((N, m)))
    U = np.ascontiguousarray(U)
    np.testing.assert_array_equal(hydro.deim_oversampled(H.dev(U), n_s), ooff.deim_oversampled(U, n_s))


def test_fom_snapshots_pod_sns_deim_pipeline():
    prob = W.sedov_like(41, 2, (9, 7), (0.0, 0.0), (0.9, 0.7), delta=0.08, e_floor=1e-2,
                        vmode="uniform", vscale=0.1, name="offline")
    rng = np.random.default_rng(41)
    prob.e[:] = 1.0 + 0.5 * rng.random(prob.e.shape)
    m = prob.mesh
    bc = ofom.bc_dofs_box(m)
    prob.v.reshape(-1)[bc] = 0.0
    ctx = H.context(prob)
    f = hydro.Fom(ctx, bc)
    x, v, e, g = H.dev(prob.x), H.dev(prob.v), H.dev(prob.e), H.dev(prob.gamma)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    import oracle
    dt = 0.2 * oracle.force(prob)["dt"]
    v_os = v.clone()
    snaps = []
    vh = torch.empty_like(v)
    for _ in range(6):   # snapshots: every half stage and every full step
        f.step(x, v, e, g, visc, cfl, dt, cg_tol=1e-14, cg_max_iter=2000)
        f.stage_state(v_half=vh)
        snaps += [(vh - v_os).reshape(-1).clone(), (v - v_os).reshape(-1).clone()]
    S = torch.stack(snaps).contiguous()          # [ns][N_V]
    Phi_g, sg = hydro.pod(S, eps=0.9999)
    Phi_o, so = ooff.pod(S.cpu().numpy(), eps=0.9999)
    assert Phi_g.shape == Phi_o.shape
    _sig_close(sg, so)
    k = Phi_g.shape[1]
    # SNS: the force basis is M_V Phi_v, column by column through the device mass
    # operator, against the oracle's assembled M_V on the oracle basis
    MV = ofom.mass_v(m)
    F_g = torch.stack([f.mass_v(Phi_g[:, c].contiguous().reshape(m.dim, m.n_nodes)).reshape(-1)
                       for c in range(k)], dim=1).contiguous()
    F_o = np.stack([np.concatenate([MV @ Phi_o[c0 * m.n_nodes:(c0 + 1) * m.n_nodes, c]
                                    for c0 in range(m.dim)]) for c in range(k)], axis=1)
    good = so[:k] >= 1e-3 * so[0]
    np.testing.assert_allclose(F_g.cpu().numpy()[:, good], F_o[:, good],
                               atol=1e-8 * np.abs(F_o).max())
    # DEIM on the SNS basis: the same sampled rows (restricted to the well-separated modes)
    kk = int(good.sum())
    np.testing.assert_array_equal(hydro.deim(F_g[:, :kk].contiguous()),
                                  ooff.deim(np.ascontiguousarray(F_o[:, :kk])))


def test_pod_degenerate_cases():
    """One snapshot: k = 1 and Phi = s / |s| (sign: the 1x1 eigenvector is +1); a zero
    snapshot set: k = 0; DEIM of a square orthonormal basis selects every row once."""
    rng = np.random.default_rng(12)
    s = rng.standard_normal(1001)
    Phi, sig = hydro.pod(H.dev(s[None, :].copy()), eps=0.9999)
    assert Phi.shape == (1001, 1)
    np.testing.assert_allclose(Phi.cpu().numpy()[:, 0], s / np.linalg.norm(s), rtol=1e-13)
    np.testing.assert_allclose(sig[0], np.linalg.norm(s), rtol=1e-13)
    Phi0, _ = hydro.pod(H.dev(np.zeros((3, 50))), eps=0.9999)
    assert Phi0.shape[1] == 0
    Q, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    idx = hydro.deim(H.dev(np.ascontiguousarray(Q)))
    assert sorted(idx.tolist()) == list(range(12))
    np.testing.assert_array_equal(idx, ooff.deim(np.ascontiguousarray(Q)))


@pytest.mark.parametrize("N,m,s", [(5_000, 8, 8), (50_001, 40, 1_337), (200_000, 40, 9_999),
                                   (3_000, 40, 32)])
def test_gappy_pinv_matches_oracle(N, m, s):
    """hydro_gappy_pinv (CholQR2 on the GPU) against the oracle's library pseudo-inverse
    (numpy SVD pinv, oracle.rom.offline_projectors' step) of the same sampled rows of a seeded
    orthonormal basis; also P (U[rows]) = I."""
    rng = np.random.default_rng(N + m)
    U = np.linalg.qr(rng.standard_normal((N, m)))[0]
    rows = np.sort(rng.choice(N, s, replace=False)).astype(np.int64)
    P = hydro.gappy_pinv(H.dev(U), rows).cpu().numpy()
    ref = np.linalg.pinv(U[rows])
    scale = np.abs(ref).max()
    assert np.abs(P - ref).max() <= 1e-11 * scale
    if s >= m:
        assert np.abs(P @ U[rows] - np.eye(m)).max() <= 1e-11
    else:   # wide sample: the minimum-norm right inverse
        assert np.abs(U[rows] @ P - np.eye(s)).max() <= 1e-11


def test_offline_projectors_gpu_vs_oracle():
    """The four offline operators of a small C4-shaped batch: GPU (hydro.offline_projectors)
    against oracle.rom.offline_projectors."""
    from oracle import rom as orom
    batch = W.c4(n_sample=6, B=3, small_mesh=True)
    got = [t.cpu().numpy() for t in H.gpu_offline_ops(batch)]
    want = orom.offline_projectors(batch)
    for g, w, what in zip(got, want, ("P_v", "P_e", "C_xv", "c_x")):
        assert g.shape == w.shape, what
        assert np.abs(g - w).max() <= 1e-11 * max(np.abs(w).max(), 1e-300), what


def test_pod_eps_one_rank_deficient():
    """eps = 1 on a rank-deficient, non-zero snapshot set (near-duplicate snapshots): the GPU
    POD keeps the numerical rank (DESIGN R31), like the oracle, with an orthonormal basis --
    no noise directions reach the CholQR pass."""
    rng = np.random.default_rng(31)
    r, ns, N = 5, 20, 80_001
    A = rng.standard_normal((N, r))
    S = (A @ rng.standard_normal((r, ns))).T
    S = np.ascontiguousarray(np.concatenate([S, S[:3] * (1 + 1e-15)]))
    Phi_g, sg = hydro.pod(H.dev(S), eps=1.0)
    Phi_o, so = ooff.pod(S, eps=1.0)
    assert Phi_g.shape[1] == Phi_o.shape[1] == r
    P = Phi_g.cpu().numpy()
    assert np.abs(P.T @ P - np.eye(r)).max() <= 1e-12
    assert np.abs(P @ (P.T @ S.T) - S.T).max() <= 1e-10 * np.abs(S).max()

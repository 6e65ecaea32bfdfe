"""Input-generator pins (-m "not gpu"): lattice/dof counts against PAPER Table 1,
the Gresho profile against PAPER Sec. 6.1.1, SplitMix64 against its reference."""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_splitmix64_reference_outputs():
    got = [hex(int(z)) for z in W.splitmix64(0, 3)]
    want = [hex(int(s, 16)) for s in GOLD["splitmix64"]["seed0_first"]]
    assert got == want
    u = W.uniform01(123, 10000)
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.01


@pytest.mark.parametrize("prob", ["gresho", "sedov", "taylor_green", "triple_point"])
def test_P13_table1_dof_counts(prob):
    """P13: PAPER Table 1 N_V and N_E from the lattice generator."""
    t = GOLD["table1_dofs"][prob]
    d = t["dim"]
    m = W.lattice_mesh(d, t["k"], 2 * t["k"], t["shape"], (0.0,) * d, (1.0,) * d)
    assert m.N_V == t["N_V"] and m.N_E == t["N_E"]


def test_config_sizes():
    """SURVEY 8 sizes table for C0-C3."""
    for name, (E, nodes, NV, NE) in {"c0": (64, 289, 578, 256),
                                     "c1": (65536, 263169, 526338, 262144)}.items():
        p = W.config(name)
        assert (p.mesh.n_elem, p.mesh.n_nodes, p.mesh.N_V, p.mesh.N_E) == (E, nodes, NV, NE)


def test_P12_gresho_profile():
    """P12: |v|(0.2) = 1, p(0) = 5, p(r >= 0.4) = 3 + 4 ln 2, continuity (reading R7)."""
    g = GOLD["gresho"]
    assert W.gresho_vphi(np.array([0.2]))[0] == g["vphi_r02"]
    assert W.gresho_pressure(np.array([0.0]))[0] == g["p_r0"]
    assert abs(W.gresho_pressure(np.array([0.5]))[0] - g["p_outer"]) < 1e-15
    for r0 in (0.2, 0.4):
        lo = W.gresho_pressure(np.array([r0 - 1e-12]))[0]
        hi = W.gresho_pressure(np.array([r0 + 1e-12]))[0]
        assert abs(lo - hi) < 1e-9
    p = W.config("c1")
    vmag = np.sqrt((p.v ** 2).sum(axis=0))
    assert 0.999 < vmag.max() <= 1.0 and p.visc is False


def test_sedov_spike_and_perturbation():
    p = W.small("c2")
    h = p.mesh.h
    assert p.e[0, 0] == 0.25 / (h[0] * h[1] * h[2])
    assert (p.e[1:] == 1e-6).all()
    bnd = W.boundary_nodes(p.mesh)
    ref = W.lattice_mesh(3, 2, 4, p.mesh.shape, p.mesh.lo, p.mesh.hi)
    assert np.array_equal(p.mesh.x0[:, bnd], ref.x0[:, bnd])
    dx = np.abs(p.mesh.x0 - ref.x0)
    assert dx[:, ~bnd].max() <= 0.05 * max(h) + 1e-15 and dx[:, ~bnd].max() > 0


def test_gll_lattice_is_affine_for_q3():
    """Nodes inside elements sit at Gauss-Lobatto points (uniform lattice = affine mesh)."""
    m = W.lattice_mesh(3, 3, 6, (2, 1, 1), (0, 0, 0), (2.0, 1.0, 1.0))
    xs = np.unique(m.x0[0])
    s5 = math.sqrt(5)
    want = [0, (5 - s5) / 10, (5 + s5) / 10, 1, 1 + (5 - s5) / 10, 1 + (5 + s5) / 10, 2]
    assert np.allclose(xs, want, atol=1e-15)


def test_c4_small_batch_structure():
    b = W.c4(n_sample=5, B=4, small_mesh=True)
    m = b.base.mesh
    assert np.all(np.diff(b.sample_elems) > 0) and np.all(np.isin(b.sample_elems, b.closure_elems))
    # closure completeness: every element touching an S0 node is in the closure
    s0n = np.zeros(m.n_nodes, bool)
    s0n[m.elem_nodes[b.sample_elems].ravel()] = True
    touching = np.nonzero(s0n[m.elem_nodes].any(axis=1))[0]
    assert np.array_equal(touching, b.closure_elems)
    assert np.allclose(b.Phi_x.T @ b.Phi_x, np.eye(40), atol=1e-12)
    assert b.e_os.shape == (b.closure_elems.size * m.ne, 4)

"""GPU parity of the slab-sharded force (paper_2104_11404_b200/shard.py) with
the library on every shard: one process, the ranks' hydro contexts built on their local
(renumbered) slabs, the halo messages handed over in memory instead of through
torch.distributed (one GPU here; the distributed exchange itself is covered with gloo in
tests/test_shard.py), the gather / fixed-order accumulate / scatter by hydro_index_copy_add.
Bars: F.1 at every shard's nodes within 1e-11 of the single-domain oracle, equal bits on
every shard sharing a node, F^T.w within 1e-12, min over shards of dt bit-identical."""
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
from paper_2104_11404_b200.shard import ShardPlan, ShardedForce  # noqa: E402


def _problem(dim):
    if dim == 2:
        return W.sedov_like(91, 2, (13, 9), (0.0, 0.0), (1.3, 0.9), delta=0.08, e_floor=1e-2,
                            vmode="uniform", vscale=0.1, name="sh2")
    return W.sedov_like(92, 3, (5, 4, 3), (0.0, 0.0, 0.0), (0.5, 0.4, 0.3), delta=0.08,
                        e_floor=1e-2, vmode="radial", vscale=0.3, name="sh3")


@pytest.mark.parametrize("dim,world", [(2, 2), (2, 3), (2, 5), (3, 2), (3, 4)])
def test_sharded_force_loopback_matches_oracle(oracle_lib, dim, world):
    prob = _problem(dim)
    m = prob.mesh
    ref = oracle_lib.force(prob)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    shards = []
    for r in range(world):
        plan = ShardPlan.build(m.elem_nodes, world, r)
        ctx = hydro.HydroContext(m.dim, m.k, m.nq, H.dev(plan.elem_nodes, torch.int32),
                                 H.dev(plan.local_view(m.x0)), H.dev(m.rho0[plan.e0:plan.e1]))
        sf = ShardedForce(plan, ctx)
        F1, FTw, dt = sf.local(H.dev(plan.local_view(prob.x)), H.dev(plan.local_view(prob.v)),
                               H.dev(prob.e[plan.e0:plan.e1]), H.dev(prob.gamma[plan.e0:plan.e1]),
                               visc, cfl)
        shards.append((plan, sf, F1, FTw, dt))
    sends = {r: sf.pack(F1) for r, (plan, sf, F1, FTw, dt) in enumerate(shards)}
    for r, (plan, sf, F1, FTw, dt) in enumerate(shards):
        sf.combine(F1, {t: sends[t][r] for t in plan.peers})
    torch.cuda.synchronize()
    dt = min(float(s[4].item()) for s in shards)
    assert H.dt_bitwise(dt, ref["dt"])
    seen = {}
    for plan, sf, F1, FTw, _ in shards:
        F1h = F1.cpu().numpy()
        H.assert_close(F1h, ref["F1"][:, plan.nodes], ref["F1mag"][:, plan.nodes], H.TOL_ASSEMBLED,
                       f"rank {plan.rank} F1")
        H.assert_close(FTw.cpu().numpy(), ref["FTw"][plan.e0:plan.e1], ref["FTwmag"][plan.e0:plan.e1],
                       H.TOL_LOCAL, f"rank {plan.rank} FTw")
        for j, n in enumerate(plan.nodes):
            if n in seen:
                assert np.array_equal(seen[n], F1h[:, j])
            else:
                seen[n] = F1h[:, j].copy()
    assert len(seen) == m.n_nodes


def test_index_copy_add():
    rng = np.random.default_rng(3)
    src = rng.standard_normal((3, 50))
    dst = rng.standard_normal((3, 40))
    si, di = rng.permutation(50)[:20], rng.permutation(40)[:20]
    d = H.dev(dst.copy())
    hydro.index_copy_add(20, 3, H.dev(src), 50, H.dev(si, torch.int64), d, 40, H.dev(di, torch.int64), True)
    ref = dst.copy()
    ref[:, di] += src[:, si]
    np.testing.assert_array_equal(d.cpu().numpy(), ref)
    hydro.index_copy_add(20, 3, H.dev(src), 50, H.dev(si, torch.int64), d, 40, None, False)
    ref[:, :20] = src[:, si]
    np.testing.assert_array_equal(d.cpu().numpy(), ref)

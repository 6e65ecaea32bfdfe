"""The slab-sharded force (paper_2104_11404_b200/shard.py) on CPU: the plan
(every element on exactly one rank, consistent renumbering, symmetric halo lists) and the
N > 1 exchange with gloo at world sizes 2 and 3 -- each rank's local F.1 / F^T.w / dt come
from the oracle on its slab (the library kernel needs a GPU; tests/test_gpu_shard.py runs it),
the halo sum and the dt all-reduce are the product code.  Bars: F.1 at every rank's nodes
within 1e-11 of the single-domain oracle (magnitude-scaled), identical bits on every rank
sharing a node, F^T.w rows equal to the oracle's, dt bit-identical."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2104_11404_b200.shard import ShardPlan, ShardedForce, slab_ranges  # noqa: E402


def _prob():
    return W.sedov_like(81, 2, (7, 5), (0.0, 0.0), (0.7, 0.5), delta=0.08, e_floor=1e-2,
                        vmode="uniform", vscale=0.1, name="shard")


def test_slab_ranges_cover_once():
    for n, w in [(35, 1), (35, 2), (35, 3), (35, 8), (4, 4), (3, 5)]:
        r = slab_ranges(n, w)
        assert len(r) == w and r[0][0] == 0 and r[-1][1] == n
        assert all(a <= b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(w - 1))
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_plan_consistency(world):
    m = _prob().mesh
    plans = [ShardPlan.build(m.elem_nodes, world, r) for r in range(world)]
    assert sum(p.e1 - p.e0 for p in plans) == m.n_elem
    for p in plans:
        np.testing.assert_array_equal(p.nodes[p.elem_nodes], m.elem_nodes[p.e0:p.e1])
        assert np.all(np.diff(p.nodes) > 0)
        for t, (sidx, pos) in p.peers.items():
            q = plans[t]
            np.testing.assert_array_equal(p.nodes[sidx], q.nodes[q.peers[p.rank][0]])  # same order
            np.testing.assert_array_equal(p.iface[pos], sidx)
        covered = np.zeros(p.nodes.size, bool)
        for sidx, _ in p.peers.values():
            covered[sidx] = True
        np.testing.assert_array_equal(np.nonzero(covered)[0], p.iface)
    if world == 1:
        assert plans[0].iface.size == 0 and not plans[0].peers


def _cpu_index_op(n, dim, src, ld_src, src_idx, dst, ld_dst, dst_idx, add):
    si = torch.arange(n) if src_idx is None else src_idx
    di = torch.arange(n) if dst_idx is None else dst_idx
    s = src.reshape(dim, ld_src)
    d = dst.reshape(dim, ld_dst)
    for c in range(dim):
        if add:
            d[c, di] = d[c, di] + s[c, si]
        else:
            d[c, di] = s[c, si]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    prob = _prob()
    plan = ShardPlan.build(prob.mesh.elem_nodes, world, rank)

    def local_eval(x, v, e, gamma, visc, cfl, w=None):
        el = np.arange(plan.e0, plan.e1, dtype=np.int32)
        out = oracle.force(prob, elist=el)
        return (torch.as_tensor(plan.local_view(out["F1"])),
                torch.as_tensor(np.ascontiguousarray(out["FTw"][plan.e0:plan.e1])),
                torch.tensor([out["dt"]], dtype=torch.float64))
    sf = ShardedForce(plan, device=torch.device("cpu"), local_eval=local_eval, index_op=_cpu_index_op)
    F1, FTw, dt = sf.force(None, None, None, None, None, None)
    q.put((rank, plan.nodes, F1.numpy(), FTw.numpy(), float(dt.item())))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_force_gloo(oracle_lib, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prob = _prob()
    ref = oracle_lib.force(prob)
    from tests.gpu_helpers import assert_close, TOL_ASSEMBLED
    seen = {}
    rows = []
    for rank, nodes, F1, FTw, dt in res:
        assert np.float64(dt).tobytes() == np.float64(ref["dt"]).tobytes()
        assert_close(F1, ref["F1"][:, nodes], ref["F1mag"][:, nodes], TOL_ASSEMBLED, f"rank {rank} F1")
        rows.append(FTw)
        for j, n in enumerate(nodes):           # every rank holding a node has the same bits
            if n in seen:
                assert np.array_equal(seen[n], F1[:, j]), (rank, n)
            else:
                seen[n] = F1[:, j].copy()
    np.testing.assert_array_equal(np.concatenate(rows), ref["FTw"])

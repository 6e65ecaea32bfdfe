"""Slab-sharded full-order force evaluation over several GPUs: one process per
GPU, the elements split into contiguous index ranges (slabs of the lattice), each rank
evaluating F.1, F^T.w and dt on its own elements with its own hydro context, then

* F.1: ONE halo sum over the H1 nodes its slab shares with other ranks.  Every rank sharing a
  node receives the other ranks' partial sums at that node and adds all of them, its own
  included, in ascending rank order -- so every rank ends with the same bits at every shared
  node, independent of message arrival order (F.1 is a global N_V vector);
* dt: one all-reduce(min) of a single double -- exact, so the global dt is bit-identical to
  a single-GPU evaluation;
* F^T.w: element-local, no exchange.

The gather / accumulate / scatter steps run in the library (hydro_index_copy_add); the
messages go through torch.distributed point-to-point operations (NCCL over NVLink on a GPU
node, gloo in the CPU tests, where the tests substitute both the local evaluation and the
index operations).  Host-side setup (the plan) is plain Python: it runs once per mesh.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

import numpy as np


def slab_ranges(n_elem: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous element ranges [e0, e1) of near-equal size, rank order = index order (the
    workloads number elements lattice-wise, so a range is a slab, up to one partial layer)."""
    if world <= 0:
        raise ValueError("world must be positive")
    base, extra = divmod(n_elem, world)
    out, e0 = [], 0
    for r in range(world):
        e1 = e0 + base + (1 if r < extra else 0)
        out.append((e0, e1))
        e0 = e1
    return out


@dataclass
class ShardPlan:
    """Rank `rank`'s share of a mesh and its halo lists.

    nodes:      global ids of the rank's H1 nodes, ascending (local node i <-> nodes[i])
    elem_nodes: [n_local_elem][ND] element-to-node table renumbered to local nodes
    iface:      local indices of the nodes shared with at least one other rank, ascending
                global id (the halo accumulator's row order)
    peers:      for every other rank t sharing nodes: (send_idx, pos) -- send_idx the local
                indices of nodes_rank & nodes_t in ascending global id (the order both sides
                use for the message), pos their rows in `iface`"""
    rank: int
    world: int
    e0: int
    e1: int
    nodes: np.ndarray
    elem_nodes: np.ndarray
    iface: np.ndarray
    peers: Dict[int, Tuple[np.ndarray, np.ndarray]] = field(default_factory=dict)

    @staticmethod
    def build(elem_nodes: np.ndarray, world: int, rank: int) -> "ShardPlan":
        en = np.asarray(elem_nodes)
        ranges = slab_ranges(en.shape[0], world)
        node_sets = [np.unique(en[a:b]) for a, b in ranges]
        e0, e1 = ranges[rank]
        mine = node_sets[rank]
        local_en = np.searchsorted(mine, en[e0:e1]).astype(np.int32)
        peers = {}
        shared_any = np.zeros(mine.size, dtype=bool)
        for t in range(world):
            if t == rank:
                continue
            common = np.intersect1d(mine, node_sets[t], assume_unique=True)
            if common.size:
                idx = np.searchsorted(mine, common)
                peers[t] = idx
                shared_any[idx] = True
        iface = np.nonzero(shared_any)[0].astype(np.int64)
        plan_peers = {t: (idx.astype(np.int64), np.searchsorted(iface, idx).astype(np.int64))
                      for t, idx in peers.items()}
        return ShardPlan(rank, world, e0, e1, mine.astype(np.int64), local_en, iface, plan_peers)

    def local_view(self, a: np.ndarray) -> np.ndarray:
        """The rank's rows of a global [dim][n_nodes] nodal array."""
        return np.ascontiguousarray(a[:, self.nodes])


class ShardedForce:
    """F.1 (assembled across ranks), F^T.w (local rows) and the global dt for one rank.

    ctx: the rank's hydro.HydroContext built on plan.elem_nodes and the local x0/rho0.
    local_eval / index_op: overridable for the CPU tests (the defaults are the library's force
    evaluation and hydro_index_copy_add); messages always go through torch.distributed."""

    def __init__(self, plan: ShardPlan, ctx=None, device=None, group=None,
                 local_eval: Optional[Callable] = None, index_op: Optional[Callable] = None):
        import torch
        self.plan, self.ctx, self.group = plan, ctx, group
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dim = None if ctx is None else ctx.dim
        self._local_eval = local_eval or self._lib_eval
        self._index_op = index_op or self._lib_index_op
        to = lambda a: torch.as_tensor(a, dtype=torch.int64, device=self.device)  # noqa: E731
        self.iface = to(plan.iface)
        self.peers = {t: (to(s), to(p)) for t, (s, p) in plan.peers.items()}
        self.self_pos = to(np.arange(plan.iface.size, dtype=np.int64))

    # -- library defaults
    def _lib_eval(self, x, v, e, gamma, visc, cfl, w=None):
        return self.ctx.force_full(x, v, e, gamma, visc, cfl, w=w)

    @staticmethod
    def _lib_index_op(n, dim, src, ld_src, src_idx, dst, ld_dst, dst_idx, add):
        from . import hydro
        hydro.index_copy_add(n, dim, src, ld_src, src_idx, dst, ld_dst, dst_idx, add)

    # -- the three halo steps
    def pack(self, F1) -> Dict[int, "object"]:
        """Per peer t: this rank's partial F.1 at the nodes shared with t, [dim][n_t]."""
        import torch
        dim, ld = F1.shape
        out = {}
        for t, (sidx, _) in self.peers.items():
            buf = torch.empty((dim, sidx.numel()), dtype=F1.dtype, device=F1.device)
            self._index_op(sidx.numel(), dim, F1, ld, sidx, buf, sidx.numel(), None, False)
            out[t] = buf
        return out

    def combine(self, F1, received: Dict[int, "object"]):
        """F1 (in place) at the interface nodes := sum over the sharing ranks, ascending rank,
        of their partials (received[t] for peers, F1 itself for this rank)."""
        import torch
        dim, ld = F1.shape
        n_if = self.iface.numel()
        if n_if == 0:
            return F1
        acc = torch.zeros((dim, n_if), dtype=F1.dtype, device=F1.device)
        for t in sorted(list(received) + [self.plan.rank]):
            if t == self.plan.rank:
                self._index_op(n_if, dim, F1, ld, self.iface, acc, n_if, self.self_pos, True)
            else:
                pos = self.peers[t][1]
                self._index_op(pos.numel(), dim, received[t], pos.numel(), None, acc, n_if, pos, True)
        self._index_op(n_if, dim, acc, n_if, None, F1, ld, self.iface, False)
        return F1

    def exchange(self, sends: Dict[int, "object"]) -> Dict[int, "object"]:
        import torch
        import torch.distributed as dist
        recv = {t: torch.empty_like(b) for t, b in sends.items()}
        ops = []
        for t in sorted(sends):
            ops.append(dist.P2POp(dist.isend, sends[t], t, group=self.group))
            ops.append(dist.P2POp(dist.irecv, recv[t], t, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return recv

    def local(self, x, v, e, gamma, visc, cfl, w=None):
        """This rank's slab only: (partial F1 at its nodes, FTw of its elements, slab dt)."""
        return self._local_eval(x, v, e, gamma, visc, cfl, w)

    def force(self, x, v, e, gamma, visc, cfl, w=None):
        """(F1 assembled over all ranks at this rank's nodes, FTw of its elements, global dt)."""
        F1, FTw, dt = self.local(x, v, e, gamma, visc, cfl, w)
        if self.plan.world > 1:
            recv = self.exchange(self.pack(F1))
            self.combine(F1, recv)
            dt = self.reduce_dt(dt)
        return F1, FTw, dt

    def reduce_dt(self, dt):
        """Global min of the per-rank dt (exact); NaN on every rank if any rank's dt is NaN
        (the single-GPU rule, DESIGN R15), without relying on how a backend orders NaN."""
        import torch
        import torch.distributed as dist
        nan = torch.isnan(dt).to(dt.dtype)
        dist.all_reduce(nan, op=dist.ReduceOp.MAX, group=self.group)
        d = torch.where(torch.isnan(dt), torch.full_like(dt, float("inf")), dt)
        dist.all_reduce(d, op=dist.ReduceOp.MIN, group=self.group)
        return torch.where(nan > 0, torch.full_like(d, float("nan")), d)

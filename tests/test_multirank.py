"""The N>1 path of bench.py (replicas only: DESIGN "Multi-GPU") on CPU with gloo,
world_size 2: every rank's time is reduced to the slowest rank's, and the whole-job value
counts every rank's units (weak scaling)."""
from __future__ import annotations

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 10.0 + 5.0 * rank                   # rank 1 is the slow replica
    dist.barrier()
    m = bench.max_over_ranks(ms, torch.device("cpu"), world)
    v = bench.whole_job_value(1_000_000, m, world)
    q.put((rank, m, v))
    dist.destroy_process_group()


def test_max_over_ranks_and_whole_job_value_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, v in res:
        assert m == 15.0                      # max over ranks, seen by every rank
        assert v == pytest.approx(2 * 1_000_000 / 15e-3)


def test_single_rank_is_identity():
    import bench
    assert bench.max_over_ranks(3.5, None, 1) == 3.5
    assert bench.whole_job_value(100, 2.0, 1) == pytest.approx(100 / 2e-3)

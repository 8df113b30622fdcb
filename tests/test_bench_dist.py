"""bench.py's multi-rank host logic (replicas, max-over-ranks timing) on CPU with
world_size 2 over gloo -- no GPU involved."""
import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    local_ms = [12.5, 7.25][rank] * 20      # rank 0 is the slow one
    tot = bench.max_over_ranks(local_ms, dist)
    q.put((rank, tot, bench.replica_value(world, 1 << 28, tot / 20)))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_replica_value_gloo():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank sees the slowest rank's time; value counts both replicas' keys
    assert [r[1] for r in res] == [250.0, 250.0]
    assert res[0][2] == pytest.approx(2 * (1 << 28) / 12.5e-3 / 1e9)


def test_single_rank_is_identity():
    import bench
    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.replica_value(1, 1 << 28, 6.7) == pytest.approx((1 << 28) / 6.7e-3 / 1e9)

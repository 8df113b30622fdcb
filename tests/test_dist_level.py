"""The multi-GPU SquareSort level's host logic (paper_2407_14801_b200.dist, SURVEY
8(e), row f3) on CPU: world_size 2 and 3 over gloo, the local sorts replaced by
numpy's (the exchange, sampling, counting and ownership logic is what is tested).
The pivots must equal the CPU oracle's sampler on the global level (sampling from
the level input, L9); the concatenated output must be the sorted input."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _np_sort(t):
    import torch
    t.copy_(torch.from_numpy(np.sort(t.numpy())))


def _inputs(kind, n, world):
    rng = np.random.default_rng(n + world)
    if kind == "uniform":
        keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    elif kind == "dups":
        keys = rng.integers(0, 40, n, dtype=np.uint64).astype(np.uint32)
    elif kind == "equal":
        keys = np.full(n, 7, np.uint32)
    else:  # sorted, with the max value
        keys = np.sort(rng.integers(0, 2**32, n, dtype=np.uint64)).astype(np.uint32)
        keys[-1] = 0xFFFFFFFF
    cuts = np.sort(rng.integers(0, n + 1, world - 1))
    return keys, np.concatenate([[0], cuts, [n]])


def _worker(rank, world, port, kind, n, q):
    import torch
    import torch.distributed as dist
    from paper_2407_14801_b200 import dist as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    keys, cuts = _inputs(kind, n, world)
    block = torch.from_numpy(keys[cuts[rank]:cuts[rank + 1]].copy())
    out, info = D.sort_distributed_u32(block, 11, dist, local_sort=_np_sort)
    q.put((rank, out.numpy().copy(), info))
    dist.barrier()
    dist.destroy_process_group()


def _run(kind, n, world):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, kind, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted((q.get(timeout=240) for _ in ps), key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("kind,n,world", [("uniform", 40000, 2), ("uniform", 30011, 3), ("dups", 20000, 2),
                                          ("equal", 5000, 2), ("sorted", 12345, 3)])
def test_distributed_level(kind, n, world):
    import oracle as O
    keys, _ = _inputs(kind, n, world)
    res = _run(kind, n, world)
    out = np.concatenate([r[1] for r in res])
    assert np.array_equal(out, np.sort(keys))  # globally sorted, a permutation
    infos = [r[2] for r in res]
    for inf in infos[1:]:  # every rank agrees on the level
        assert np.array_equal(inf["pivots"], infos[0]["pivots"])
        assert inf["round"] == infos[0]["round"] and inf["owner_first_bucket"] == infos[0]["owner_first_bucket"]
    # the pivots are the single-GPU sampler's: the oracle's level sampler on the global input
    m = O.ceil_sqrt(n)
    D = keys.astype(np.uint64).copy()
    for a in range(0, n, m):
        D[a:a + m] = np.sort(D[a:a + m])
    P, r, deg = O.sample_pivots(O.root_key(11), keys, D)
    assert np.array_equal(infos[0]["pivots"].astype(np.uint64), P)
    assert infos[0]["round"] == r and infos[0]["degenerate"] == deg
    # ownership: contiguous bucket ranges, ranks in key order, balanced within one bucket's size
    sizes = [len(x[1]) for x in res]
    assert sum(sizes) == n
    if kind == "uniform":
        assert max(sizes) - min(sizes) <= 16 * m

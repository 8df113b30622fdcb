"""The multi-GPU level (paper_2407_14801_b200.dist) through its CUDA path: one rank,
NCCL, the library's sorts (this pool gives one GPU per run; the multi-rank exchange
logic is covered on CPU by tests/test_dist_level.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_distributed_level_one_rank_nccl():
    import torch.distributed as dist
    import oracle as O
    from paper_2407_14801_b200 import dist as D
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        for n in (1 << 20, 300007):
            keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
            out, info = D.sort_distributed_u32(torch.from_numpy(keys).cuda(), 5, dist)
            assert np.array_equal(out.cpu().numpy(), np.sort(keys))
            m = O.ceil_sqrt(n)
            Dm = keys.astype(np.uint64).copy()
            for a in range(0, n, m):
                Dm[a:a + m] = np.sort(Dm[a:a + m])
            P, r, deg = O.sample_pivots(O.root_key(5), keys, Dm)
            assert np.array_equal(info["pivots"].astype(np.uint64), P) and info["round"] == r
    finally:
        dist.destroy_process_group()

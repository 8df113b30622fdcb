"""SquareSort's level across G GPUs: one process per GPU,
torch.distributed (NCCL over NVLink/NVSwitch) for the exchange.

The level is Alg 1 with the columns distributed: rank r holds a
contiguous block of the n keys (its columns), and
  1. sorts them on its GPU (the column pass; libsquaresort's SquareSort);
  2. all ranks draw the SAME sample positions of the global level input from the
     counter-based RNG (sq_draw_positions; sampled from the level
     input as on one GPU, L9), each rank fills in the positions it owns and one
     all-reduce(SUM) assembles every round's m-1 candidates; every rank sorts them
     (libsquaresort) and takes the first round that is strictly increasing with
     its smallest pivot above the global minimum (all-reduce MIN), else the last
     round, degenerate -- identical pivots on every rank;
  3. counts every bucket in its sorted block (bucket(x) = #{P < x} + [x in P],
     L2/L4) and all-gathers the G x m counts: the buckets are cut into G
     contiguous ranges of nearly equal key counts, range q owned by rank q;
  4. SkewTranspose becomes an all-to-allv: rank r's keys of range q are one
     contiguous run of its sorted block; the runs arrive in rank order (= column
     order, the order Alg 3 gives inside a bucket);
  5. sorts what it received (the bucket pass; libsquaresort).
The output is globally sorted and distributed by contiguous key range: rank q
holds the keys of buckets [b_q, b_{q+1}), in order, and ranks are in key order.

`local_sort` defaults to the library's GPU sort (CUDA tensors, fails loudly
without the extension); tests of the host logic on CPU (gloo) pass their own.
"""
from __future__ import annotations

import math

import numpy as np


def _ceil_sqrt(n: int) -> int:
    r = math.isqrt(n)
    return r if r * r == n else r + 1


def _default_local_sort(t):
    import paper_2407_14801_b200 as sq
    return sq.sort_u32(t)


def _i64(t):
    """uint32 tensor -> int64 values (through an int32 view: torch's uint32 support is partial)."""
    import torch
    return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF


def level_pivots(block, off: int, n: int, seed: int, gmin: int, dist, local_sort=None, cap: int = 32):
    """(pivots [m-1] uint32 tensor, round, degenerate) of the global level (step 2).
    block: this rank's UNSORTED keys (the level input, L9), global positions [off, off+len);
    gmin: the level's minimum."""
    import torch
    import paper_2407_14801_b200 as sq
    local_sort = local_sort or _default_local_sort
    m = _ceil_sqrt(n)
    npv = m - 1
    dev = block.device
    node = sq.root_key(seed)
    pos_all = sq.draw_positions(node, cap, npv, n).astype(np.int64)  # [cap, m-1], the same on every rank
    for r in range(cap):
        pos = torch.from_numpy(pos_all[r]).to(dev)
        mine = (pos >= off) & (pos < off + block.numel())
        cand = torch.zeros(npv, dtype=torch.int64, device=dev)
        cand[mine] = _i64(block)[(pos[mine] - off)]
        dist.all_reduce(cand, op=dist.ReduceOp.SUM)  # every position is owned by exactly one rank
        c32 = cand.to(torch.int32).view(torch.uint32).contiguous() if npv else cand.to(torch.int32).view(torch.uint32)
        if npv:
            local_sort(c32)
        c64 = _i64(c32)
        ok = npv == 0 or (bool((c64[1:] > c64[:-1]).all().item()) and int(c64[0].item()) > gmin)
        if ok or r == cap - 1:
            return c32, r, 0 if ok else 1
    raise AssertionError("unreachable")


def bucket_bounds(sorted_block, pivots):
    """Positions of the m-1 bucket boundaries in a sorted block (equal-pivot rule L4):
    boundary j (1..m-1) = #{x < P[j-1]}, or #{x <= P[j-1]} when P[j-1] repeats P[j-2]."""
    import torch
    if pivots.numel() == 0:
        return torch.zeros(0, dtype=torch.int64, device=sorted_block.device)
    flip = -2**31  # unsigned order == signed order after flipping the sign bit
    b = sorted_block.view(torch.int32) ^ flip
    p = pivots.view(torch.int32) ^ flip
    left = torch.searchsorted(b, p, right=False)
    right = torch.searchsorted(b, p, right=True)
    dup = torch.zeros(p.shape, dtype=torch.bool, device=p.device)
    dup[1:] = p[1:] == p[:-1]
    return torch.where(dup, right, left).to(torch.int64)


def owner_ranges(counts: np.ndarray, world: int) -> np.ndarray:
    """First bucket of every rank's range (length world+1): contiguous ranges of the
    m buckets with nearly equal global key counts.  counts: [world, m] per-rank counts."""
    tot = counts.sum(axis=0)
    cum = np.concatenate([[0], np.cumsum(tot)])
    n = int(cum[-1])
    b = [0]
    for q in range(1, world):
        # first bucket boundary at or past q*n/world
        b.append(int(np.searchsorted(cum, q * n / world, side="left")))
    b.append(len(tot))
    b = np.maximum.accumulate(np.minimum(np.array(b), len(tot)))
    return b


def sort_distributed_u32(block, seed: int, dist, local_sort=None):
    """Globally sort the uint32 keys spread over the ranks of `dist` (torch.distributed,
    initialised).  block: this rank's keys (CUDA uint32 tensor with NCCL; CPU with
    gloo and an injected local_sort).  Returns (this rank's sorted key range, info)."""
    import torch
    local_sort = local_sort or _default_local_sort
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = block.device
    sizes = torch.tensor([block.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    all_sizes = [int(x.item()) for x in all_sizes]
    n, off = sum(all_sizes), sum(all_sizes[:rank])
    if n < 2:
        out = block.clone()
        if out.numel():
            local_sort(out)
        return out, {"n": n, "m": 1, "round": 0, "degenerate": 0, "owner_first_bucket": [0] * (world + 1)}
    # 1. the column pass: this rank's columns, sorted on its GPU (the input stays for sampling)
    work = block.clone()
    if work.numel():
        local_sort(work)
    # 2. pivots, sampled from the level input (L9); min(D) = the smallest column head
    gm = torch.tensor([int(_i64(work[:1]).item()) if work.numel() else 2**32], dtype=torch.int64, device=dev)
    dist.all_reduce(gm, op=dist.ReduceOp.MIN)
    pivots, rnd, deg = level_pivots(block, off, n, seed, int(gm.item()), dist, local_sort)
    # 3. bucket counts, all-gathered; owner ranges
    bounds = bucket_bounds(work, pivots)
    edges = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), bounds,
                       torch.tensor([work.numel()], dtype=torch.int64, device=dev)])
    counts = (edges[1:] - edges[:-1]).contiguous()
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    cmat = np.stack([c.cpu().numpy() for c in all_counts])
    first = owner_ranges(cmat, world)
    # 4. SkewTranspose as an all-to-allv: rank q receives every rank's run of its buckets
    e = edges.cpu().numpy()
    send_splits = [int(e[first[q + 1]] - e[first[q]]) for q in range(world)]
    recv_splits = [int(cmat[r, first[rank]:first[rank + 1]].sum()) for r in range(world)]
    recv = torch.empty(sum(recv_splits), dtype=torch.int32, device=dev)  # uint32 bits in int32 transport
    dist.all_to_all_single(recv, work.view(torch.int32), recv_splits, send_splits)
    recv = recv.view(torch.uint32)
    # 5. the bucket pass: this rank's buckets, sorted on its GPU
    if recv.numel():
        local_sort(recv)
    info = {"n": n, "m": _ceil_sqrt(n), "round": rnd, "degenerate": deg,
            "owner_first_bucket": [int(x) for x in first], "send": send_splits, "recv": recv_splits,
            "pivots": _i64(pivots).cpu().numpy()}
    return recv, info

"""Out-of-core SquareSort (the analog of the paper's external-sorting
experiment: 64-bit integers in a memory-mapped file): sorting n keys
that live in host memory -- a numpy array or np.memmap, possibly larger than the
GPU's memory -- with one SquareSort level whose columns and buckets are streamed
through the GPU.  Every sort is libsquaresort's; this module only moves data.

The level (Alg 1) on the host array A of n keys, device budget B keys:
  * pivots: m-1 with m = ceil(sqrt(n)), drawn by the library's
    counter-based RNG at the root node from the level input A (L9) before A is
    touched; the round rule of P:297-305 / S:94 (strictly increasing, smallest
    above min(D); degenerate after 32 rounds) is applied after the column pass;
  * column pass: A is cut into columns of C = B keys (a rectangular level: the
    GPU's column is as long as its memory allows); every column is copied to the
    GPU, sorted there and copied back in place (sq_sort_*_host_batch: copies of
    column i+1 and i-1 overlap the sort of column i);
  * bucket positions: per column, the position of every bucket boundary by binary
    search in the sorted column (bucket(x) = #{P < x} + [x in P], L2/L4);
  * SkewTranspose + bucket pass: consecutive buckets are packed into groups of at
    most C keys (units, reading L24); for every group the runs of all columns are
    gathered in column order (the order Alg 3 writes), sorted on the
    GPU and written to their final place in `out`.  A single-value bucket (the
    equal-pivot rule) is copied; a bucket larger than C recurses.
"""
from __future__ import annotations

import math

import numpy as np


def _ceil_sqrt(n: int) -> int:
    r = math.isqrt(n)
    return r if r * r == n else r + 1


def _sort_host(x: np.ndarray, seed: int):
    import paper_2407_14801_b200 as sq
    if x.dtype == np.uint32:
        sq.sort_u32_host(x, seed)
    else:
        sq.sort_u64_host(x, seed)


def _boundaries(col: np.ndarray, piv: np.ndarray) -> np.ndarray:
    """Positions of the m-1 bucket boundaries in a sorted column (L4 equal-pivot rule)."""
    left = np.searchsorted(col, piv, side="left")
    right = np.searchsorted(col, piv, side="right")
    dup = np.zeros(len(piv), bool)
    dup[1:] = piv[1:] == piv[:-1]
    return np.where(dup, right, left)


def sort_external(keys: np.ndarray, out: np.ndarray | None = None, seed: int = 0,
                  budget_keys: int | None = None, stats: dict | None = None) -> np.ndarray:
    """Sort the uint32 or uint64 `keys` (host memory; left as sorted columns) into `out`
    (host memory, same dtype and length; allocated when None).  `budget_keys`: keys of
    one column / bucket group held on the GPU (default: an eighth of the free device memory,
    in keys: the sort's scratch and the batch's three buffers fit beside it)."""
    import paper_2407_14801_b200 as sq
    if keys.dtype not in (np.uint32, np.uint64):
        raise TypeError("keys must be uint32 or uint64")
    n = int(keys.size)
    if out is None:
        out = np.empty_like(keys)
    if out.dtype != keys.dtype or out.size != n:
        raise ValueError("out must match keys in dtype and length")
    if stats is None:
        stats = {}
    stats.setdefault("levels", 0)
    stats["levels"] += 1
    if budget_keys is None:
        import torch
        free, _ = torch.cuda.mem_get_info()
        budget_keys = max(1 << 16, int(free // (keys.itemsize * 8)))
    C = max(1024, int(budget_keys))
    if n <= C:  # fits: one on-GPU SquareSort
        out[:] = keys
        if n > 1:
            _sort_host(out, seed)
        return out
    m = _ceil_sqrt(n)
    npv = m - 1
    # pivot candidates of every round, from the level input (L9), before the column pass
    node = sq.root_key(seed)
    rounds = 32
    pos = sq.draw_positions(node, rounds, npv, n).astype(np.int64)
    cand = np.ascontiguousarray(keys[pos.reshape(-1)].reshape(rounds, npv))
    # column pass: columns of C keys sorted on the GPU, in place in `keys`
    ncol = (n + C - 1) // C
    full = [keys[i * C:(i + 1) * C] for i in range(n // C)]
    if full:
        batch = sq.sort_u32_host_batch if keys.dtype == np.uint32 else sq.sort_u64_host_batch
        work = [np.ascontiguousarray(c) for c in full] if not keys.flags.c_contiguous else full
        batch(work, work, seed)
        if work is not full:
            for c, w in zip(full, work):
                c[:] = w
    if n % C:
        tail = np.ascontiguousarray(keys[(n // C) * C:])
        _sort_host(tail, seed)
        keys[(n // C) * C:] = tail
    cols = [keys[i * C:min((i + 1) * C, n)] for i in range(ncol)]
    # round selection: min(D) = the smallest column head
    gmin = min(int(c[0]) for c in cols)
    chosen, deg = rounds - 1, 1
    for r in range(rounds):
        c = cand[r].copy()
        if npv > 1:
            _sort_host(c, seed)
        cand[r] = c
        if npv == 0 or (np.all(c[1:] > c[:-1]) and int(c[0]) > gmin):
            chosen, deg = r, 0
            break
    piv = cand[chosen]  # (sorted above: the loop ends at the chosen or the last round)
    stats.setdefault("round", chosen)
    stats.setdefault("degenerate", deg)
    stats.setdefault("pivots", piv.copy())
    # bucket boundaries of every column, sizes, starts (analysis convention)
    bnd = np.stack([np.concatenate([[0], _boundaries(c, piv), [len(c)]]) for c in cols])  # [ncol, m+1]
    sizes = (bnd[:, 1:] - bnd[:, :-1]).sum(axis=0)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    single = np.zeros(m, bool)
    single[1:npv] = piv[1:] == piv[:-1]  # bucket j >= 1 with P[j-1] == P[j]: one value (L4)
    # bucket pass: groups of consecutive buckets of at most C keys
    j = 0
    stats.setdefault("groups", 0)
    while j < m:
        if sizes[j] > C and not single[j]:  # an oversize bucket: another level on it
            run = np.concatenate([c[bnd[i, j]:bnd[i, j + 1]] for i, c in enumerate(cols)])
            sort_external(run, out[starts[j]:starts[j + 1]], seed ^ (0x9E3779B97F4A7C15 * (j + 1) % 2**64),
                          C, stats)
            j += 1
            continue
        j1, tot = j, 0
        while j1 < m and (tot + sizes[j1] <= C or j1 == j) and not (sizes[j1] > C and not single[j1]):
            tot += sizes[j1]
            j1 += 1
        # SkewTranspose of the group: every column's run of buckets [j, j1), in column order
        grp = np.concatenate([c[bnd[i, j]:bnd[i, j1]] for i, c in enumerate(cols)])
        if len(grp) > 1 and not (j1 == j + 1 and single[j]):
            _sort_host(grp, seed)
        out[starts[j]:starts[j1]] = grp
        stats["groups"] += 1
        j = j1
    return out

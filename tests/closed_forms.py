"""Closed forms the oracle and the GPU path are pinned against (test code only).

These are the plain definitions of what SquareSort reaches:
  * a keys-only sort has a unique result: the ascending copy (np.sort);
  * a pairs sort is taken to be stable (L16): np.argsort(kind="stable");
  * SkewTranspose with given pivots is the stable partition of the
    column-major source by bucket(x) = #{P < x} + [x in P] (L2, L4), written
    at the bucket cursors, with buc_out[j] = buc_in[j] + size_j.
"""
import numpy as np


def bucket_ids(x, pivots):
    P = np.asarray(pivots, dtype=np.uint64)
    x = np.asarray(x, dtype=np.uint64)
    if len(P) == 0:
        return np.zeros(len(x), np.int64)
    lb = np.searchsorted(P, x, side="left")
    ub = np.searchsorted(P, x, side="right")
    return (lb + (ub > lb)).astype(np.int64)


def skew_transpose(src, pivots, k=None, buc_in=None, n=None, vals=None):
    src = np.asarray(src, dtype=np.uint64)
    n = len(src) if n is None else n
    k = len(pivots) + 1 if k is None else k
    x = src[:n]
    b = bucket_ids(x, pivots)
    sizes = np.bincount(b, minlength=k)[:k]
    if buc_in is None:
        start = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    else:
        start = np.asarray(buc_in, dtype=np.int64)
    order = np.argsort(b, kind="stable")
    bo = b[order]
    first = np.searchsorted(bo, np.arange(k), side="left")
    rank = np.arange(n) - first[bo]
    pos = start[bo] + rank
    dst = np.zeros(len(src), np.uint64)
    dst[pos] = x[order]
    dv = None
    if vals is not None:
        v = np.asarray(vals, dtype=np.uint32)[:n]
        dv = np.zeros(len(src), np.uint32)
        dv[pos] = v[order]
    return dst, dv, (start + sizes).astype(np.uint64)


def stable_pairs_sort(keys, vals):
    o = np.argsort(np.asarray(keys), kind="stable")
    return np.asarray(keys)[o], np.asarray(vals)[o]

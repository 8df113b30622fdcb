"""Out-of-core SquareSort (paper_2407_14801_b200.external, f4; the analog of the
paper's external sort of 64-bit integers in a memory-mapped file):
a host array much larger than the device budget given to the level, against
np.sort and the oracle's sampler."""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import oracle as O  # noqa: E402
from paper_2407_14801_b200 import external as E  # noqa: E402


@pytest.mark.parametrize("dt,kind,n,budget", [(np.uint32, "uniform", 1 << 22, 1 << 18),
                                              (np.uint64, "uniform", 3_000_017, 1 << 18),
                                              (np.uint32, "dups", 1 << 21, 1 << 16),
                                              (np.uint64, "binary", 1 << 20, 1 << 15)])
def test_external_sort(dt, kind, n, budget):
    rng = np.random.default_rng(n)
    if kind == "uniform":
        keys = rng.integers(0, np.iinfo(dt).max, n, dtype=dt, endpoint=True)
    elif kind == "dups":
        keys = rng.integers(0, 1000, n, dtype=np.uint64).astype(dt)
    else:
        keys = rng.integers(0, 2, n, dtype=np.uint64).astype(dt)
    want = np.sort(keys)
    a = keys.copy()
    st = {}
    out = E.sort_external(a, seed=9, budget_keys=budget, stats=st)
    assert np.array_equal(out, want)
    assert st["groups"] >= 1
    # the level's pivots are the oracle sampler's on the same input (L9 source, min(D) rule)
    m = O.ceil_sqrt(n)
    D = keys.astype(np.uint64).copy()
    for s in range(0, n, m):
        D[s:s + m] = np.sort(D[s:s + m])
    P, r, deg = O.sample_pivots(O.root_key(9), keys, D)
    assert st["round"] == r and st["degenerate"] == deg
    assert np.array_equal(st["pivots"].astype(np.uint64), P)


def test_external_sort_memmap():
    n = 1 << 21
    rng = np.random.default_rng(1)
    keys = rng.integers(0, 2**63, n, dtype=np.uint64)
    with tempfile.TemporaryDirectory() as d:
        src = np.memmap(os.path.join(d, "keys.bin"), dtype=np.uint64, mode="w+", shape=(n,))
        dst = np.memmap(os.path.join(d, "out.bin"), dtype=np.uint64, mode="w+", shape=(n,))
        src[:] = keys
        E.sort_external(src, dst, seed=3, budget_keys=1 << 17)
        assert np.array_equal(np.asarray(dst), np.sort(keys))
        del src, dst

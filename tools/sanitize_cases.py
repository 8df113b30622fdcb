"""Small sorts for compute-sanitizer runs (memcheck / racecheck / synccheck), one
tool per process: cfg1 (2^16), cfg2 (2^20) and a forced multi-level case (max
tile 512 on 2^17 keys) in each big-bucket mode, u64 with duplicates, pairs, the
counting- and merge-sort base cases, and the standalone SkewTranspose.  Every
result is checked against np.sort / the closed form.  Usage:
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py [quick]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_14801_b200 as sq  # noqa: E402
import sqinputs as S  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"


def check_u32(keys, seed):
    t = torch.from_numpy(keys).cuda()
    sq.sort_u32(t, seed)
    assert np.array_equal(t.cpu().numpy(), np.sort(keys))


cases = []
k1, _ = S.config("cfg1")
cases.append(("cfg1", lambda: check_u32(k1, 1)))
if not quick:
    k2, _ = S.config("cfg2")
    cases.append(("cfg2", lambda: check_u32(k2, 2)))
km, _ = S.generate("uniform_u32", 1 << 17, 9)


def multilevel(mode, base):
    def run():
        sq.set_max_tile(512)
        sq.set_big_bucket_mode(mode)
        sq.set_base_case(base)
        try:
            check_u32(km, 9)
        finally:
            sq.set_max_tile(0)
            sq.set_big_bucket_mode(sq.BIG_MERGE)
            sq.set_base_case(sq.BASE_BIN)
    return run


for mode in (sq.BIG_LEVEL, sq.BIG_MERGE, sq.BIG_CLUSTER):
    for base in (sq.BASE_BIN, sq.BASE_MERGE):
        cases.append((f"multilevel mode={mode} base={base}", multilevel(mode, base)))


def u64_dups():
    k, _ = S.generate("dup1000_u64", 1 << 16, 3)
    t = torch.from_numpy(k).cuda()
    sq.sort_u64(t, 3)
    assert np.array_equal(t.cpu().numpy(), np.sort(k))


def pairs():
    k, v = S.generate("perm_pairs_u32", 1 << 16, 5)
    tk, tv = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    sq.sort_pairs_u32_u32(tk, tv, 5)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(tk.cpu().numpy(), k[order]) and np.array_equal(tv.cpu().numpy(), v[order])


def skew():
    rows = cols = 256
    rng = np.random.default_rng(4)
    x = rng.integers(0, 2**32, rows * cols, dtype=np.uint64).astype(np.uint32)
    for c in range(cols):
        x[c * rows:(c + 1) * rows] = np.sort(x[c * rows:(c + 1) * rows])
    piv = np.sort(rng.choice(x, cols - 1, replace=False))
    src = torch.from_numpy(x).cuda()
    dst = torch.zeros_like(src)
    bo = sq.skew_transpose(src, dst, rows, cols, pivots=torch.from_numpy(piv).cuda())
    b = np.searchsorted(piv, x, side="right")  # bucket(x) = #{P <= x} for distinct pivots
    want = x[np.argsort(b, kind="stable")]
    assert np.array_equal(dst.cpu().numpy(), want)
    assert int(bo.cpu().numpy()[-1]) == rows * cols


cases += [("u64 duplicates", u64_dups), ("pairs", pairs), ("skew_transpose", skew)]
for name, fn in cases:
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)
print("all cases ok")

"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element, on the seeded BASELINE configs and edge cases.  Integer work, so
the bar is bit-exact everywhere."""
import numpy as np
import pytest

import oracle as O
import sqinputs as S
from tests import closed_forms as CF

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2407_14801_b200 as sq  # noqa: E402


@pytest.fixture(autouse=True)
def _reset_tile():
    sq.set_max_tile(0)
    sq.set_big_bucket_mode(sq.BIG_MERGE)
    yield
    sq.set_max_tile(0)
    sq.set_big_bucket_mode(sq.BIG_MERGE)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def to_host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def gpu_sort(keys, seed=0, vals=None):
    k = to_dev(keys)
    if vals is not None:
        v = to_dev(vals)
        sq.sort_pairs_u32_u32(k, v, seed)
        return to_host(k), to_host(v)
    if keys.dtype == np.uint32:
        sq.sort_u32(k, seed)
    else:
        sq.sort_u64(k, seed)
    return to_host(k)


def oracle_sort(keys, seed, vals=None):
    d, dv, st = O.square_sort(keys, vals, seed=seed)
    return d.astype(keys.dtype), (None if dv is None else dv)


# ---------------------------------------------------------------- configs vs oracle
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_config_vs_oracle(cfg):
    keys, _ = S.config(cfg)
    seed = S.CONFIGS[cfg][2]
    want, _ = oracle_sort(keys, seed)
    got = gpu_sort(keys, seed)
    assert got.dtype == keys.dtype and np.array_equal(got, want)


def test_cfg3_u64_duplicates_vs_oracle():
    keys, _ = S.config("cfg3")
    want, _ = oracle_sort(keys, 3)
    got = gpu_sort(keys, 3)
    assert np.array_equal(got, want)
    st = sq.get_stats()
    assert st["top_degenerate"] == 1 and st["top_round"] == 31  # 4095 draws from 1000 values


@pytest.mark.parametrize("cfg", ["cfg4_sorted", "cfg4_reverse", "cfg4_swapped", "cfg4_nonsquare"])
def test_cfg4_variants(cfg):
    keys, _ = S.config(cfg)
    got = gpu_sort(keys, 4)
    want = np.sort(keys)  # closed form: the unique ascending permutation
    assert np.array_equal(got, want)
    if cfg == "cfg4_sorted":
        assert np.array_equal(got, keys)
    if cfg == "cfg4_reverse":
        assert np.array_equal(got, keys[::-1])


def test_cfg4_scaled_vs_oracle():
    # the same recipes at 2^20, where the oracle itself runs in seconds
    for cfg in ("cfg4_sorted", "cfg4_reverse", "cfg4_swapped"):
        keys, _ = S.config(cfg, n=1 << 20)
        want, _ = oracle_sort(keys, 4)
        assert np.array_equal(gpu_sort(keys, 4), want), cfg
    keys, _ = S.config("cfg4_nonsquare", n=(1 << 20) - 12345)
    want, _ = oracle_sort(keys, 4)
    assert np.array_equal(gpu_sort(keys, 4), want)


def test_cfg5_full_size():
    keys, _ = S.config("cfg5")
    got = gpu_sort(keys, 5)
    assert np.all(got[1:] >= got[:-1])
    want = np.sort(keys)
    assert np.array_equal(got, want)
    # sampled order statistics straight from the definition (rank of out[i])
    rng = np.random.default_rng(0)
    for i in rng.integers(0, len(keys), 3):
        x = got[i]
        assert (keys < x).sum() <= i < (keys <= x).sum()


def test_cfg5p_pairs_full_size():
    keys, vals = S.config("cfg5p")
    gk, gv = gpu_sort(keys, 5, vals)
    n = len(keys)
    assert np.array_equal(gk, np.arange(n, dtype=np.uint32))
    inv = np.empty(n, np.uint32)
    inv[keys] = np.arange(n, dtype=np.uint32)  # vals_out[k] = input position of key k
    assert np.array_equal(gv, inv)


@pytest.mark.parametrize("n,card", [(1 << 18, 2**64), (200003, 1000), (70000, 3), (1 << 20, 2**40)])
def test_pairs_u64_vs_oracle(n, card):
    """u64 keys with a u32 payload (f1; P:1048's 64-bit workload): stable, against the oracle."""
    rng = np.random.default_rng(n ^ 77)
    if card == 2**64:
        keys = rng.integers(0, 2**63, n, dtype=np.uint64) * 2 + rng.integers(0, 2, n, dtype=np.uint64)
    else:
        keys = rng.integers(0, card, n, dtype=np.uint64)
    vals = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    want_k, want_v = O.square_sort(keys, vals, seed=3)[:2]
    k, v = to_dev(keys), to_dev(vals)
    sq.sort_pairs_u64_u32(k, v, 3)
    assert np.array_equal(to_host(k), want_k) and np.array_equal(to_host(v), want_v)
    ek, ev = CF.stable_pairs_sort(keys, vals)
    assert np.array_equal(want_k, ek) and np.array_equal(want_v, ev)


def test_pairs_u64_modes_and_host():
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 5000, 300001, dtype=np.uint64) << np.uint64(33)
    vals = np.arange(len(keys), dtype=np.uint32)
    ek, ev = CF.stable_pairs_sort(keys, vals)
    for mode in (sq.BIG_LEVEL, sq.BIG_MERGE, sq.BIG_CLUSTER):
        sq.set_max_tile(1024)
        sq.set_big_bucket_mode(mode)
        k, v = to_dev(keys), to_dev(vals)
        sq.sort_pairs_u64_u32(k, v, 1)
        assert np.array_equal(to_host(k), ek) and np.array_equal(to_host(v), ev), mode
    sq.set_max_tile(0)
    sq.set_big_bucket_mode(sq.BIG_MERGE)
    hk, hv = keys.copy(), vals.copy()
    sq.sort_pairs_u64_u32_host(hk, hv, 2)
    assert np.array_equal(hk, ek) and np.array_equal(hv, ev)


def test_pairs_scaled_vs_oracle():
    keys, vals = S.config("cfg5p", n=1 << 18)
    want_k, want_v = oracle_sort(keys, 5, vals)
    gk, gv = gpu_sort(keys, 5, vals)
    assert np.array_equal(gk, want_k) and np.array_equal(gv, want_v)


# ---------------------------------------------------------------- maximum sizes
def _check_sorted_perm_gpu(src, out):
    """out is non-decreasing and a permutation of src (sums of x, x^2 mod 2^64 and a
    histogram of the top byte agree); a few order statistics checked by definition."""
    a, b = src.to(torch.int64), out.to(torch.int64)
    assert bool((b[1:] >= b[:-1]).all())
    assert int(a.sum()) == int(b.sum()) and int((a * a).sum()) == int((b * b).sum())
    assert torch.equal(torch.bincount(a >> 24, minlength=256), torch.bincount(b >> 24, minlength=256))
    for i in (0, len(b) // 3, len(b) - 1):
        x = b[i]
        assert int((a < x).sum()) <= i < int((a <= x).sum())


def test_max_size_u32():
    # the documented limit n = 2^30 (4 GiB of keys)
    g = torch.Generator(device="cuda").manual_seed(30)
    src = torch.randint(0, 2**32, (1 << 30,), device="cuda", dtype=torch.int64, generator=g).to(torch.uint32)
    out = src.clone()
    sq.sort_u32(out, 30)
    _check_sorted_perm_gpu(src, out)


def test_max_size_u64():
    # the documented limit n = 2^28 for 64-bit keys (values below 2^40: int64-safe checks)
    g = torch.Generator(device="cuda").manual_seed(28)
    src = torch.randint(0, 2**40, (1 << 28,), device="cuda", dtype=torch.int64, generator=g).to(torch.uint64)
    out = src.clone()
    sq.sort_u64(out, 28)
    _check_sorted_perm_gpu(src.to(torch.int64), out.to(torch.int64))


# ---------------------------------------------------------------- edge cases
EDGE_N = [0, 1, 2, 3, 4, 5, 16, 17, 63, 64, 65, 255, 256, 257, 1000, 4095, 4096, 4097,
          32767, 32768, 32769, 65535, 65536, 65537, 100000, 250001]


@pytest.mark.parametrize("n", EDGE_N)
def test_sizes_u32(n):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(gpu_sort(keys, n), np.sort(keys))


@pytest.mark.parametrize("n", [0, 1, 5, 17, 1000, 16384, 16385, 70000])
def test_sizes_u64(n):
    rng = np.random.default_rng(n + 1)
    keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    assert np.array_equal(gpu_sort(keys, 7), np.sort(keys))


@pytest.mark.parametrize("mode", [0, 1, 2, 4])
@pytest.mark.parametrize("tile", [64, 256, 1024])
@pytest.mark.parametrize("n", [5000, 70001, 300000])
def test_forced_multilevel_vs_oracle(tile, n, mode):
    # a small on-chip tile forces the big-bucket path (merge sort or clusters, up
    # to 16 tiles) and, past it or in mode 0, SquareSort levels in columns and buckets
    sq.set_max_tile(tile)
    sq.set_big_bucket_mode(mode)
    rng = np.random.default_rng(tile * 7 + n)
    for card in (2**32, 1000, 3):
        keys = rng.integers(0, card, n, dtype=np.uint64).astype(np.uint32)
        want, _ = oracle_sort(keys, 11)
        got = gpu_sort(keys, 11)
        assert np.array_equal(got, want), card
        if card == 2**32 and n >= 16 * tile and mode == 0:
            assert sq.get_stats()["levels"] >= 2


@pytest.mark.parametrize("mode", [0, 1, 2, 4])
@pytest.mark.parametrize("tile", [64, 512])
def test_forced_multilevel_pairs_and_u64(tile, mode):
    sq.set_max_tile(tile)
    sq.set_big_bucket_mode(mode)
    rng = np.random.default_rng(tile)
    n = 50000
    k = rng.integers(0, 50, n, dtype=np.uint64).astype(np.uint32)
    v = np.arange(n, dtype=np.uint32)
    gk, gv = gpu_sort(k, 3, v)
    ek, ev = CF.stable_pairs_sort(k, v)
    assert np.array_equal(gk, ek) and np.array_equal(gv, ev)
    k64 = rng.integers(0, 2**64, n, dtype=np.uint64)
    assert np.array_equal(gpu_sort(k64, 3), np.sort(k64))


def test_special_values():
    n = 200000
    rng = np.random.default_rng(3)
    for keys in (np.full(n, 0xFFFFFFFF, np.uint32), np.zeros(n, np.uint32),
                 np.where(rng.random(n) < 0.5, 0xFFFFFFFF, 0).astype(np.uint32),
                 rng.integers(0xFFFFFFF0, 2**32, n, dtype=np.uint64).astype(np.uint32)):
        assert np.array_equal(gpu_sort(keys, 1), np.sort(keys))
    k64 = np.full(70000, 2**64 - 1, np.uint64)
    k64[::7] = 0
    assert np.array_equal(gpu_sort(k64, 1), np.sort(k64))


def test_pairs_stability_with_duplicates():
    rng = np.random.default_rng(5)
    for n, card in ((1000, 3), (100000, 100), (300000, 2**32)):
        k = rng.integers(0, card, n, dtype=np.uint64).astype(np.uint32)
        v = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        gk, gv = gpu_sort(k, 9, v)
        ek, ev = CF.stable_pairs_sort(k, v)
        assert np.array_equal(gk, ek) and np.array_equal(gv, ev)


@pytest.mark.parametrize("mode", [0, 1, 2, 4])
def test_big_bucket_modes_full_tile(mode):
    # default tiles, 2^24 keys: buckets of ~4K with a tail beyond 16K exercise each mode
    sq.set_big_bucket_mode(mode)
    keys, _ = S.config("cfg5", n=1 << 24)
    assert np.array_equal(gpu_sort(keys, 5), np.sort(keys))
    k, v = S.config("cfg5p", n=1 << 23)
    gk, gv = gpu_sort(k, 5, v)
    assert np.array_equal(gk, np.arange(len(k), dtype=np.uint32))
    assert np.array_equal(gk[gv], np.arange(len(k), dtype=np.uint32)[gv]) and np.array_equal(k[gv], gk)


def test_seed_invariance():
    keys, _ = S.config("cfg2")
    ref = gpu_sort(keys, 2)
    for seed in (0, 12345, 2**63 + 5):
        assert np.array_equal(gpu_sort(keys, seed), ref)


def test_host_entry_points():
    keys, _ = S.config("cfg2")
    h = keys.copy()
    sq.sort_u32_host(h, 2)
    assert np.array_equal(h, np.sort(keys))
    k, v = S.config("cfg5p", n=1 << 16)
    hk, hv = k.copy(), v.copy()
    sq.sort_pairs_u32_u32_host(hk, hv, 5)
    ek, ev = CF.stable_pairs_sort(k, v)
    assert np.array_equal(hk, ek) and np.array_equal(hv, ev)
    k64, _ = S.config("cfg3", n=1 << 16)
    h64 = k64.copy()
    sq.sort_u64_host(h64, 3)
    assert np.array_equal(h64, np.sort(k64))


def test_host_batch_entry_points():
    # pipelined batch: distinct inputs, a shared input, an in-place item, a ragged n
    import torch
    n = 300001
    ins = [S.generate("uniform_u32", n, s)[0] for s in (1, 2)]
    pin = [torch.empty(n, dtype=torch.uint32).pin_memory().numpy() for _ in range(4)]
    for p, a in zip(pin, ins + ins):
        np.copyto(p, a)
    outs = [np.empty(n, np.uint32) for _ in range(3)] + [pin[3]]
    sq.sort_u32_host_batch([pin[0], pin[1], pin[0], pin[3]], outs, 4)
    for o, a in zip(outs, [ins[0], ins[1], ins[0], ins[1]]):
        assert np.array_equal(o, np.sort(a))
    # a reused output keeps the last item's result
    r = np.empty(n, np.uint32)
    sq.sort_u32_host_batch([pin[0], pin[1], pin[0], pin[1]], [r, pin[2], r, pin[2]], 4)
    assert np.array_equal(r, np.sort(ins[0])) and np.array_equal(pin[2], np.sort(ins[1]))
    assert np.array_equal(pin[0], ins[0])  # inputs untouched
    k64 = [S.generate("dup1000_u64", 70001, s)[0] for s in (3, 4, 5)]
    o64 = [np.empty_like(k) for k in k64]
    sq.sort_u64_host_batch(k64, o64, 9)
    for o, a in zip(o64, k64):
        assert np.array_equal(o, np.sort(a))
    one = [np.array([7], np.uint32)]
    o1 = [np.zeros(1, np.uint32)]
    sq.sort_u32_host_batch(one, o1)
    assert o1[0][0] == 7


# ---------------------------------------------------------------- one level vs the oracle's level
@pytest.mark.parametrize("n,card", [(1 << 16, 2**32), (1 << 20, 2**32), (100003, 2**32),
                                    (1 << 16, 1000), (50000, 7)])
def test_level_intermediate_parity(n, card):
    """Pivots, accepted round, bucket ends and the post-SkewTranspose array of
    one level equal the oracle's, sampling from the level input (L9)."""
    rng = np.random.default_rng(n ^ card)
    keys = rng.integers(0, card, n, dtype=np.uint64).astype(np.uint32)
    seed = 77
    post, _, P, be, r, deg = O.level(keys, seed=seed, sample_from_input=True)
    m = O.ceil_sqrt(n)
    src = to_dev(keys)
    dst = torch.empty_like(src)
    piv = torch.empty(m - 1, dtype=torch.uint32, device="cuda")
    bend = torch.empty(m, dtype=torch.uint32, device="cuda")
    info = torch.empty(2, dtype=torch.uint32, device="cuda")
    sq.debug_level_u32(src, dst, seed, piv, bend, info)
    assert np.array_equal(to_host(piv).astype(np.uint64), P)
    assert np.array_equal(to_host(bend).astype(np.uint64), be)
    assert to_host(info).tolist() == [r, deg]
    assert np.array_equal(to_host(dst).astype(np.uint64), post)
    assert np.array_equal(to_host(src), keys)  # src untouched


# ---------------------------------------------------------------- sq_skew_transpose
def _sorted_cols(x, rows, n):
    x = x.copy()
    for a in range(0, n, rows):
        x[a:min(a + rows, n)] = np.sort(x[a:min(a + rows, n)])
    return x


def gpu_skew(src, rows, cols, pivots, k=None, n=0, buc_in=None, T=4, flags=0):
    s = to_dev(src.astype(np.uint32))
    d = torch.zeros_like(s) if len(src) else torch.zeros(1, dtype=torch.uint32, device="cuda")
    pv = to_dev(np.asarray(pivots, np.uint32)) if len(pivots) else None
    bi = to_dev(np.asarray(buc_in, np.uint32)) if buc_in is not None else None
    bo = sq.skew_transpose(s, d, rows, cols, pv, k, n, bi, None, T, flags)
    return to_host(d), to_host(bo)


@pytest.mark.parametrize("T", [4, 10, 2])
def test_cfg2_skew_transpose_check(T):
    """BASELINE config 2's SkewTranspose check: the 2^20 keys as a 1024x1024
    matrix, columns sorted, pivots from the oracle's sampler at root mix(2)."""
    keys, _ = S.config("cfg2")
    n, m = len(keys), 1024
    D = _sorted_cols(keys.astype(np.uint64), m, n)
    P, r, deg = O.sample_pivots(O.root_key(2), D, D)
    want, _, wbo = O.skew_transpose_matrix(D, m, m, P, T=T)
    got, gbo = gpu_skew(D, m, m, P, T=T)
    assert np.array_equal(got.astype(np.uint64), want)
    assert np.array_equal(gbo.astype(np.uint64), wbo)


@pytest.mark.parametrize("seed", range(12))
def test_skew_transpose_u64_random_shapes(seed):
    """sq_skew_transpose_u64 (f1) against the oracle's Alg 2 and the closed form: ragged and
    empty columns, duplicate pivots, keys above 2^32, caller cursors."""
    rng = np.random.default_rng(1000 + seed)
    rows, cols = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    n = int(rng.integers(0, rows * cols + 1))
    card = [2**64, 2**40, 50][seed % 3]
    if card == 2**64:
        x = rng.integers(0, 2**63, rows * cols, dtype=np.uint64) * 2 + 1
    else:
        x = rng.integers(0, card, rows * cols, dtype=np.uint64)
    x = _sorted_cols(x, rows, n)
    k = int(rng.integers(1, 70))
    P = np.sort(rng.choice(x[: max(n, 1)], k - 1)) if n and k > 1 else np.sort(rng.integers(0, card, k - 1, dtype=np.uint64))
    want, _, wbo = O.skew_transpose_matrix(x, rows, cols, P, k, n=n, T=int(rng.integers(2, 6)))
    dc, _, bc = CF.skew_transpose(x, P, k, n=n)
    assert (want[:n] == dc[:n]).all() and (wbo == bc).all()
    s = to_dev(x)
    d = torch.zeros_like(s)
    pv = to_dev(P.astype(np.uint64)) if k > 1 else None
    bi = None
    if seed % 2:  # caller cursors: buckets in reverse order
        sizes = bc - np.concatenate([[0], bc[:-1]]).astype(np.uint64)
        bi = np.concatenate([[0], np.cumsum(sizes[::-1])[:-1]])[::-1].astype(np.uint32)
        want, _, wbo = O.skew_transpose_matrix(x, rows, cols, P, k, n=n, buc_in=bi.astype(np.uint64))
    bo = sq.skew_transpose(s, d, rows, cols, pv, k, n, to_dev(bi) if bi is not None else None)
    assert np.array_equal(to_host(d)[:n], want[:n])
    assert np.array_equal(to_host(bo).astype(np.uint64), wbo)
    st = sq.get_stats()
    assert st["host_syncs"] == 1  # cursors scanned / checked on the device


def test_skew_transpose_bad_cursors_rejected():
    rows = cols = 64
    x = _sorted_cols(np.arange(rows * cols, dtype=np.uint64)[::-1].copy(), rows, rows * cols)
    P = np.arange(1, cols, dtype=np.uint64) * rows
    bi = np.full(cols, rows * cols - 1, np.uint32)  # every range but one leaves dst
    for dt in (np.uint32, np.uint64):
        s = to_dev(x.astype(dt))
        d = torch.zeros_like(s)
        with pytest.raises(sq.SqError) as e:
            sq.skew_transpose(s, d, rows, cols, to_dev(P.astype(dt)), cols, 0, to_dev(bi))
        assert e.value.code == 1
        assert int(to_host(d).astype(np.uint64).sum()) == 0  # nothing was written


def test_skew_transpose_special_case_is_transpose():
    m = 300  # one item of every bucket per column -> plain transpose
    src = np.array([c + r * m for c in range(m) for r in range(m)], np.uint64)
    P = np.array([j * m for j in range(1, m)], np.uint64)
    got, _ = gpu_skew(src, m, m, P)
    assert np.array_equal(got.reshape(m, m), src.reshape(m, m).T.astype(np.uint32))


@pytest.mark.parametrize("case", range(40))
def test_skew_transpose_random_shapes(case):
    rng = np.random.default_rng(1000 + case)
    rows = int(rng.integers(1, 3000))
    cols = int(rng.integers(1, 300))
    n = int(rng.integers(0, rows * cols + 1)) if case % 3 == 0 else rows * cols
    k = int(rng.choice([1, 2, cols, cols + 1, max(1, cols // 2), int(rng.integers(1, 5000))]))
    card = int(rng.choice([3, 100, 2**32]))
    x = rng.integers(0, card, rows * cols, dtype=np.uint64)
    if case % 5 == 0:
        x[rng.random(len(x)) < 0.3] = 0xFFFFFFFF
    x = _sorted_cols(x, rows, n)
    if case % 2:
        P = np.sort(rng.choice(x[:max(n, 1)], k - 1)) if k > 1 else np.zeros(0, np.uint64)
    else:
        P = np.sort(rng.integers(0, card, k - 1, dtype=np.uint64))
    buc_in = None
    if case % 4 == 1:  # explicit cursors, buckets laid out in reverse order
        _, _, bc = CF.skew_transpose(x, P, k, n=n)
        sizes = bc - np.concatenate([[0], bc[:-1]]).astype(np.uint64)
        buc_in = np.concatenate([[0], np.cumsum(sizes[::-1])[:-1]])[::-1].astype(np.uint64)
    want, _, wbo = O.skew_transpose_matrix(x, rows, cols, P, k, n=n, buc_in=buc_in)
    got, gbo = gpu_skew(x, rows, cols, P, k=k, n=n, buc_in=buc_in, T=int(rng.integers(2, 12)))
    assert np.array_equal(got[:n].astype(np.uint64), want[:n])
    assert np.array_equal(gbo.astype(np.uint64), wbo)


def test_skew_transpose_validate_flag():
    x = np.array([3, 1, 2, 4], np.uint64)  # column 0 unsorted
    with pytest.raises(sq.SqError) as e:
        gpu_skew(x, 2, 2, [2], flags=sq.SQ_FLAG_VALIDATE)
    assert e.value.code == 4
    x = np.array([1, 3, 2, 4], np.uint64)
    with pytest.raises(sq.SqError) as e:
        gpu_skew(x, 2, 2, [3, 2], flags=sq.SQ_FLAG_VALIDATE)
    assert e.value.code == 4
    got, bo = gpu_skew(x, 2, 2, [2, 3], flags=sq.SQ_FLAG_VALIDATE)
    assert got.tolist() == [1, 2, 3, 4] and bo.tolist() == [1, 2, 4]


# ---------------------------------------------------------------- signed / IEEE keys (L25)
@pytest.mark.parametrize("dt", ["int32", "int64", "float32", "float64"])
@pytest.mark.parametrize("n", [1000, 300007])
def test_signed_and_float_keys(dt, n):
    rng = np.random.default_rng(31)
    npdt = np.dtype(dt)
    if npdt.kind == "i":
        info = np.iinfo(npdt)
        x = rng.integers(info.min, info.max, n, dtype=npdt, endpoint=True)
        x[:3] = [info.min, info.max, 0]
        x[3:600] = x[3]  # a run of duplicates
    else:
        x = (rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)).astype(npdt)
        u = np.uint32 if npdt.itemsize == 4 else np.uint64
        w = npdt.itemsize * 8
        specials = np.array([np.inf, -np.inf, 0.0, -0.0, np.finfo(npdt).tiny, -np.finfo(npdt).tiny], npdt)
        nans = np.array([(1 << w) - 1, (1 << (w - 1)) - 1, (1 << (w - 1)) | 1], u).view(npdt)
        x[: len(specials)] = specials
        x[len(specials): len(specials) + 3] = nans
    # expected: the oracle's total-order key, sorted, mapped back (the definition)
    k = O.total_order_key(x)
    want = O.from_total_order_key(np.sort(k), npdt)
    t = torch.from_numpy(x.copy()).cuda()
    getattr(sq, "sort_" + {"int32": "i32", "int64": "i64", "float32": "f32", "float64": "f64"}[dt])(t, 7)
    got = t.cpu().numpy()
    u = np.uint32 if npdt.itemsize == 4 else np.uint64
    assert np.array_equal(got.view(u), want.view(u))


def test_concurrent_calls_two_threads():
    # the header allows concurrent calls on different streams with disjoint buffers
    # (per-thread library state); ctypes releases the GIL during the calls
    import threading
    rng = np.random.default_rng(41)
    arrs = [rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32) for n in (3_000_001, 1_500_007)]
    outs, errs = [None, None], []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                t = torch.from_numpy(arrs[i]).cuda()
                for _ in range(3):
                    w = t.clone()
                    sq.sort_u32(w, i, stream=s)
                s.synchronize()
                outs[i] = w.cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs
    for a, o in zip(arrs, outs):
        assert np.array_equal(o, np.sort(a))


# ---------------------------------------------------------------- counting-sort clusters (mode 3)
@pytest.mark.parametrize("lg", [24, 26])
def test_bincluster_mode_uniform(lg):
    # m = 4096 / 8192: buckets of 16K-128K keys go to clusters of 2, 4, 8 counting-sort tiles
    sq.set_big_bucket_mode(sq.BIG_BINCLUSTER)
    keys = S.uniform_u32(1 << lg, 40 + lg)
    assert np.array_equal(gpu_sort(keys, 3), np.sort(keys))


def test_bincluster_mode_skewed_falls_back_to_next_level():
    # heavy values inside buckets make a value range larger than one tile: those
    # buckets go to the next SquareSort level (oversize), the sort stays exact
    sq.set_big_bucket_mode(sq.BIG_BINCLUSTER)
    n = 1 << 26
    rng = np.random.default_rng(77)
    keys = S.uniform_u32(n, 77)
    heavy = rng.integers(0, 2**32, 200, dtype=np.uint64).astype(np.uint32)
    pos = rng.choice(n, 200 * 12000, replace=False)
    keys[pos] = np.repeat(heavy, 12000)
    assert np.array_equal(gpu_sort(keys, 9), np.sort(keys))
    assert sq.get_stats()["oversize_keys"] > 0


def test_bincluster_mode_level_state_vs_oracle():
    # the whole sort at cfg-like shape against the oracle itself (2^22: m = 2048)
    sq.set_big_bucket_mode(sq.BIG_BINCLUSTER)
    keys = S.uniform_u32(1 << 22, 12)
    want, _ = oracle_sort(keys, 12)
    assert np.array_equal(gpu_sort(keys, 12), want)


# ---------------------------------------------------------------- value-split big buckets (mode 4)
@pytest.mark.parametrize("lg", [24, 26])
def test_split_mode_uniform(lg):
    # m = 4096 / 8192: inner buckets beyond one CTA are sorted as value ranges
    sq.set_big_bucket_mode(sq.BIG_SPLIT)
    keys = S.uniform_u32(1 << lg, 50 + lg)
    assert np.array_equal(gpu_sort(keys, 3), np.sort(keys))
    k64 = S.stream(60 + lg, 1 << (lg - 2))
    assert np.array_equal(gpu_sort(k64, 3), np.sort(k64))


def test_split_mode_heavy_values_halve_ranges():
    # heavy values inside buckets overflow a value range: the range is halved (and
    # re-read) down to one-value ranges written as copies; the sort stays exact
    sq.set_big_bucket_mode(sq.BIG_SPLIT)
    n = 1 << 26
    rng = np.random.default_rng(78)
    keys = S.uniform_u32(n, 78)
    heavy = rng.integers(0, 2**32, 100, dtype=np.uint64).astype(np.uint32)
    pos = rng.choice(n, 100 * 30000, replace=False)
    keys[pos] = np.repeat(heavy, 30000)
    assert np.array_equal(gpu_sort(keys, 9), np.sort(keys))
    # narrow ranges: values clustered near a few points inside wide buckets
    keys = S.uniform_u32(n, 79)
    keys[: n // 4] = (keys[: n // 4] % 64) + np.uint32(123456789)
    assert np.array_equal(gpu_sort(keys, 9), np.sort(keys))


def test_split_mode_vs_oracle():
    sq.set_big_bucket_mode(sq.BIG_SPLIT)
    keys = S.uniform_u32(1 << 22, 13)
    want, _ = oracle_sort(keys, 13)
    assert np.array_equal(gpu_sort(keys, 13), want)
    sq.set_max_tile(256)
    keys = S.uniform_u32(300001, 14)
    want, _ = oracle_sort(keys, 14)
    assert np.array_equal(gpu_sort(keys, 14), want)

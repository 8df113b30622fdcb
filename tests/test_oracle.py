"""Pins for the CPU oracle: each oracle function is checked against
something other than itself -- SPEC.md's hand-traced examples, closed forms,
brute force on tiny inputs, published RNG test vectors, and invariants.
All `-m "not gpu"`."""
import itertools
import math

import numpy as np
import pytest

import oracle as O
from tests import closed_forms as CF

GAMMA = 0x9E3779B97F4A7C15
M64 = 2**64 - 1


# ------------------------------------------------------------------ RNG
def test_mix_is_splitmix64(golden):
    sm = golden["splitmix64"]
    for i, h in enumerate(sm["seed0"]):
        assert O.mix((i * GAMMA) & M64) == int(h, 16)
    for i, d in enumerate(sm["seed1234567"]):
        assert O.mix((1234567 + i * GAMMA) & M64) == int(d)


def test_index_closed_form():
    for n in (1, 2, 3, 1000, 2**32 - 1, 2**40 + 7):
        assert O.index(0, n) == 0
        assert O.index(M64, n) == n - 1
        assert O.index(2**63, n) == n // 2
    rng = np.random.default_rng(5)
    for _ in range(200):
        d = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        n = int(rng.integers(1, 2**40))
        assert O.index(d, n) == (d * n) >> 64


def test_draw_and_child_compose_mix():
    k = 0x0123456789ABCDEF
    assert O.draw(k, 3, 77) == O.mix(k ^ O.mix((3 << 32) | 77))
    assert O.child_key(k, 1, 5) == O.mix(k ^ O.mix(11))
    assert O.child_key(k, 0, 5) == O.mix(k ^ O.mix(10))
    assert O.root_key(9) == O.mix(9)


def test_index_uniform_chi2():
    key = O.root_key(1)
    n = 10
    counts = np.zeros(n)
    N = 20000
    for i in range(N):
        counts[O.index(O.draw(key, 0, i), n)] += 1
    chi2 = ((counts - N / n) ** 2 / (N / n)).sum()
    assert chi2 < 30  # 9 dof; p ~ 4e-4


# ------------------------------------------------------------------ column layout
def test_column_layout_spec(golden):
    for ex in golden["column_layout"]:
        m, c, e = O.column_layout(ex["n"])
        assert m == ex["m"], ex["cite"]
        assert c.tolist() == ex["col"], ex["cite"]
        assert e.tolist() == ex["colEnd"], ex["cite"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 15, 16, 17, 255, 256, 257, 2**20 - 1, 2**20,
                               2**20 + 1, 2**26 - 12345, 2**28, 2**27, 2**40 + 3, 2**62 - 1])
def test_ceil_sqrt_exact(n):
    r = math.isqrt(n)
    want = r if r * r == n else r + 1
    assert O.ceil_sqrt(n) == want


def test_column_layout_tiles_range():
    for n in list(range(1, 300)) + [2**26 - 12345, 2**27]:
        m, c, e = O.column_layout(n)
        assert m == math.isqrt(n - 1) + 1
        assert c[0] == 0 and e[-1] == n
        assert (c[1:] == e[:-1]).all()
        assert ((e - c) <= m).all()


def test_layout_of_nonsquare_configs():
    # 4' = 8190 full + 1 of 4039 + 1 empty; 5p = 11584 full + 5504 + empty
    for n, m, full, part in ((2**26 - 12345, 8192, 8190, 4039), (2**27, 11586, 11584, 5504)):
        mm, c, e = O.column_layout(n)
        L = e - c
        assert mm == m and (L == m).sum() == full and L[full] == part and L[full + 1] == 0


# ------------------------------------------------------------------ simple_sort / MergeSort
def test_simple_sort_examples():
    assert O.simple_sort([3, 1, 2]).tolist() == [1, 2, 3]
    assert O.simple_sort(np.zeros(0, np.uint64)).tolist() == []
    x = np.random.default_rng(7).integers(0, 2**64, 16, dtype=np.uint64)
    assert (O.simple_sort(x) == np.sort(x)).all()


def test_simple_sort_stable():
    rng = np.random.default_rng(3)
    k = rng.integers(0, 4, 50)
    v = np.arange(50)
    d, dv = O.simple_sort(k, v)
    ek, ev = CF.stable_pairs_sort(k, v)
    assert (d == ek).all() and (dv == ev).all()


def test_merge_sort():
    rng = np.random.default_rng(4)
    for n in (0, 1, 2, 3, 17, 1000):
        x = rng.integers(0, 50, n, dtype=np.uint64)
        assert (O.merge_sort(x) == np.sort(x)).all()


# ------------------------------------------------------------------ bucket cursors
def _cols(n, rows):
    c = np.minimum(np.arange(0, n + rows, rows)[: (n + rows - 1) // rows], n)
    return c, np.minimum(c + rows, n)


def test_initial_bucket_cursors_spec(golden):
    for ex in golden["initial_bucket_cursors"]:
        c, e = _cols(len(ex["D"]), ex["rows"])
        buc = O.initial_bucket_cursors(ex["D"], c, e, ex["pivots"])
        assert buc.tolist() == ex["buc"], ex["cite"]


def _random_instance(rng, ncols, rows, k, ncard=None, n=None, dup_pivots=False):
    """Sorted columns (ragged last) and k-1 non-decreasing pivots."""
    n = ncols * rows if n is None else n
    card = ncard or 2**32
    x = rng.integers(0, card, n, dtype=np.uint64)
    c, e = _cols(n, rows) if rows else (np.zeros(0, np.int64), np.zeros(0, np.int64))
    c, e = c[:ncols], e[:ncols]
    for a, b in zip(c, e):
        x[a:b] = np.sort(x[a:b])
    if dup_pivots:
        pool = x if len(x) else np.arange(3, dtype=np.uint64)
        P = np.sort(rng.choice(pool, k - 1, replace=True)) if k > 1 else np.zeros(0, np.uint64)
    else:
        P = np.sort(rng.integers(0, card, k - 1, dtype=np.uint64))
    return x, c, e, P


def test_initial_bucket_cursors_closed_form():
    rng = np.random.default_rng(11)
    for trial in range(300):
        ncols = int(rng.integers(1, 20))
        rows = int(rng.integers(1, 20))
        k = int(rng.integers(1, 25))
        x, c, e, P = _random_instance(rng, ncols, rows, k, ncard=int(rng.integers(2, 60)),
                                      dup_pivots=bool(trial % 2))
        buc = O.initial_bucket_cursors(x, c, e, P, k)
        _, _, bo = CF.skew_transpose(x, P, k)
        sizes = bo - np.concatenate([[0], bo[:-1]]).astype(np.uint64)
        want = np.concatenate([[0], np.cumsum(sizes)[:-1]])
        assert (buc == want).all()


# ------------------------------------------------------------------ SkewTranspose
def test_naive_skew_transpose_spec(golden):
    for ex in golden["naive_skew_transpose"]:
        c, e = _cols(len(ex["src"]), ex["rows"])
        d, _, col, buc = O.naive_skew_transpose(ex["src"], c, e, ex["pivots"], ex["buc"])
        assert d.tolist() == ex["dst"], ex["cite"]
        assert buc.tolist() == ex["buc_after"], ex["cite"]
        assert col.tolist() == ex["col_after"], ex["cite"]


def test_skew_transpose_spec(golden):
    for ex in golden["skew_transpose"]:
        c, e = _cols(len(ex["src"]), ex["rows"])
        d, _, col, buc = O.skew_transpose(ex["src"], c, e, ex["pivots"], ex["buc"],
                                          T=ex["threshold"])
        assert d.tolist() == ex["dst"], ex["cite"]
        assert buc.tolist() == ex["buc_after"], ex["cite"]


def test_bucket_ranges_spec(golden):
    # bucket j = [buc_after[j-1], buc_after[j]) with buc_after[-1] = 0
    for ex in golden["bucket_ranges"]:
        b = [0] + ex["buc_after"]
        assert [[b[j], b[j + 1]] for j in range(len(ex["buc_after"]))] == ex["ranges"]


@pytest.mark.parametrize("T", [2, 3, 4, 10])
def test_skew_transpose_equals_naive_and_closed_form(T):
    rng = np.random.default_rng(100 + T)
    for trial in range(150):
        m = int(rng.integers(1, 24))
        k = max(1, int(rng.choice([m, m + 1, m - 1, m // 2])))
        rows = int(rng.integers(1, 24))
        n = int(rng.integers(0, m * rows + 1))
        x, c, e, P = _random_instance(rng, m, rows, k, n=n, ncard=int(rng.integers(2, 1000)),
                                      dup_pivots=bool(trial % 3 == 0))
        if len(c) < m:  # trailing empty columns
            c = np.concatenate([c, np.full(m - len(c), n)])
            e = np.concatenate([e, np.full(m - len(e), n)])
        buc = O.initial_bucket_cursors(x, c, e, P, k)
        v = rng.integers(0, 2**32, len(x), dtype=np.uint64).astype(np.uint32)
        d1, dv1, col1, b1 = O.naive_skew_transpose(x, c, e, P, buc, vals=v)
        d2, dv2, col2, b2 = O.skew_transpose(x, c, e, P, buc, T=T, vals=v)
        assert (d1 == d2).all() and (b1 == b2).all() and (col1 == col2).all()
        assert (dv1 == dv2).all()
        dc, dvc, bc = CF.skew_transpose(x, P, k, vals=v)
        assert (d1 == dc).all() and (b1 == bc).all() and (dv1 == dvc).all()
        # cursor conservation and bijection
        assert (col1 == e).all()
        assert int((b1 - buc).sum()) == len(x)


def test_skew_transpose_is_matrix_transpose_in_special_case():
    # when every sorted column holds exactly one item of every bucket,
    # SkewTranspose is the ordinary transpose.  Column c = {c + r*m}, pivots j*m.
    m = 13
    src = np.array([c + r * m for c in range(m) for r in range(m)], np.uint64)
    P = np.array([j * m for j in range(1, m)], np.uint64)
    c, e = _cols(m * m, m)
    buc = O.initial_bucket_cursors(src, c, e, P)
    d, _, _, _ = O.skew_transpose(src, c, e, P, buc, T=4)
    assert (d.reshape(m, m) == src.reshape(m, m).T).all()


def test_skew_transpose_k1_is_copy():
    rng = np.random.default_rng(9)
    x, c, e, P = _random_instance(rng, 7, 5, 1)
    d, _, _, b = O.skew_transpose(x, c, e, P, [0], T=2)
    assert (d == x).all() and b.tolist() == [len(x)]


def test_split_balance_invariant():
    # |k - l| <= 1 is kept by the split; checked arithmetically.
    def walk(l, k, T):
        assert abs(k - l) <= 1
        if l < T or k < T:
            return
        l2, k2 = l // 2, k // 2
        for a, b in ((l2, k2), (l - l2, k2), (l2, k - k2), (l - l2, k - k2)):
            walk(a, b, T)
    for m in range(1, 200):
        walk(m, m, 2)


def test_skew_transpose_matrix_entry():
    rng = np.random.default_rng(21)
    for trial in range(60):
        rows = int(rng.integers(1, 30))
        cols = int(rng.integers(1, 30))
        n = int(rng.integers(0, rows * cols + 1))
        k = int(rng.integers(1, 40))
        x, _, _, P = _random_instance(rng, cols, rows, k, n=rows * cols,
                                      ncard=int(rng.integers(2, 200)), dup_pivots=trial % 2 == 0)
        for cc in range(cols):
            a, b = min(cc * rows, n), min((cc + 1) * rows, n)
            x[a:b] = np.sort(x[a:b])
        d, _, bo = O.skew_transpose_matrix(x, rows, cols, P, k, n=n, T=int(rng.integers(2, 6)))
        dc, _, bc = CF.skew_transpose(x, P, k, n=n)
        assert (d[:n] == dc[:n]).all() and (bo == bc).all()
        # explicit cursors: buckets placed in reverse order
        sizes = bc - np.concatenate([[0], bc[:-1]]).astype(np.uint64)
        bi = np.concatenate([[0], np.cumsum(sizes[::-1])[:-1]])[::-1].astype(np.uint64)
        d2, _, bo2 = O.skew_transpose_matrix(x, rows, cols, P, k, n=n, buc_in=bi)
        dc2, _, bc2 = CF.skew_transpose(x, P, k, n=n, buc_in=bi)
        assert (d2[:n] == dc2[:n]).all() and (bo2 == bc2).all()


# ------------------------------------------------------------------ pivot sampling
def test_sample_pivots_spec_examples():
    # [1,2,3,4] as 2 columns -> one pivot in {2,3,4}
    for s in range(50):
        P, r, deg = O.sample_pivots(O.root_key(s), [1, 2, 3, 4], [1, 2, 3, 4])
        assert len(P) == 1 and P[0] in (2, 3, 4) and deg == 0
    # all-equal -> degenerate after the cap
    P, r, deg = O.sample_pivots(7, [5, 5, 5, 5], [5, 5, 5, 5], cap=32)
    assert deg == 1 and r == 31 and P.tolist() == [5]


def test_sample_pivots_invariants_and_round_rule():
    rng = np.random.default_rng(2)
    n = 400
    x = rng.permutation(n).astype(np.uint64) + 10
    m = O.ceil_sqrt(n)
    D = x.copy()
    for a in range(0, n, m):
        D[a:a + m] = np.sort(D[a:a + m])
    for s in range(30):
        node = O.root_key(s)
        P, r, deg = O.sample_pivots(node, x, D)
        assert deg == 0 and len(P) == m - 1
        assert (np.diff(P.astype(np.int64)) > 0).all() and P[0] > D.min()
        assert set(P.tolist()) <= set(x.tolist())
        # the accepted round is the FIRST round passing both checks:
        for rr in range(r + 1):
            cand = np.sort([x[O.index(O.draw(node, rr, i), n)] for i in range(m - 1)])
            ok = (np.diff(cand.astype(np.int64)) > 0).all() and cand[0] > D.min()
            assert ok == (rr == r)
            if rr == r:
                assert (cand == P).all()


@pytest.mark.parametrize("cap", [32, 5, 1])
def test_sample_pivots_degenerate_keeps_last_round(cap):
    # S:94 / L8: after `cap` failed rounds the pivots are degenerate and round cap-1's
    # sorted candidates are kept.  Low cardinality (400 keys over 3 values) makes every
    # round fail (m-1 = 19 draws cannot be strictly increasing); the kept set must be
    # round cap-1's draw, recomputed from the RNG spec (a different round's draw differs).
    rng = np.random.default_rng(21)
    n = 400
    x = rng.integers(0, 3, n).astype(np.uint64) + 5
    m = O.ceil_sqrt(n)
    D = x.copy()
    for a in range(0, n, m):
        D[a:a + m] = np.sort(D[a:a + m])
    for s in range(10):
        node = O.root_key(s)
        P, r, deg = O.sample_pivots(node, x, D, cap=cap)
        assert deg == 1 and r == cap - 1
        rounds = [np.sort([x[O.index(O.draw(node, rr, i), n)] for i in range(m - 1)]) for rr in range(cap)]
        assert (P == rounds[cap - 1]).all()
        if cap > 1:  # the rounds differ, so keeping another round would be caught
            assert any((rounds[rr] != rounds[cap - 1]).any() for rr in range(cap - 1))


def test_mean_rounds_closed_form():
    # Distinct keys: a round succeeds iff the m-1 positions are distinct and avoid the
    # minimum: p = prod_{i=0}^{m-2} (n-1-i)/n; E[rounds] = 1/p  (<= e^2).
    n = 2500
    m = O.ceil_sqrt(n)
    p = np.prod([(n - 1 - i) / n for i in range(m - 1)])
    x = np.arange(n, dtype=np.uint64)
    D = x.copy()
    rounds = []
    for s in range(1500):
        _, r, deg = O.sample_pivots(O.root_key(s), x, D, cap=64)
        assert deg == 0
        rounds.append(r + 1)
    rounds = np.array(rounds, float)
    mu, sd = 1 / p, math.sqrt(1 - p) / p
    assert abs(rounds.mean() - mu) < 4 * sd / math.sqrt(len(rounds))
    assert rounds.mean() <= math.e**2


# ------------------------------------------------------------------ SquareSort
def test_square_sort_spec(golden):
    d, _, _ = O.square_sort([42])
    assert d.tolist() == [42]
    d, _, _ = O.square_sort(np.arange(100, 0, -1))
    assert d.tolist() == list(range(1, 101))


@pytest.mark.parametrize("n", range(0, 10))
def test_square_sort_all_permutations(n):
    for perm in itertools.permutations(range(n)):
        d, _, _ = O.square_sort(np.array(perm, np.uint64), cutoff=4, seed=n)
        assert d.tolist() == list(range(n))


@pytest.mark.parametrize("n", range(5, 10))
def test_square_sort_all_ternary(n):
    for t in itertools.product(range(3), repeat=n):
        d, _, _ = O.square_sort(np.array(t, np.uint64), cutoff=4, seed=1)
        assert d.tolist() == sorted(t)


def test_square_sort_all_binary_12():
    for bits in range(1 << 12):
        t = [(bits >> i) & 1 for i in range(12)]
        d, _, _ = O.square_sort(np.array(t, np.uint64), cutoff=4, seed=bits)
        assert d.tolist() == sorted(t)


@pytest.mark.parametrize("cutoff,T,src", [(16, 4, False), (4, 2, True), (100, 10, False),
                                          (1000, 10, True)])
def test_square_sort_random_vs_sorted_copy(cutoff, T, src):
    rng = np.random.default_rng(cutoff)
    for n in (17, 100, 1000, 12345):
        for card in (2, 50, 2**32, 2**64):
            x = rng.integers(0, card, n, dtype=np.uint64) if card < 2**64 else \
                rng.integers(0, 2**63, n, dtype=np.uint64) * 2 + 1
            d, _, st = O.square_sort(x, cutoff=cutoff, threshold=T, seed=n,
                                     sample_from_input=src)
            assert (d == np.sort(x)).all()


def test_square_sort_pairs_stable():
    rng = np.random.default_rng(8)
    for n, card in ((1000, 7), (5000, 2**32), (3000, 40)):
        k = rng.integers(0, card, n, dtype=np.uint64)
        v = np.arange(n, dtype=np.uint32)
        d, dv, _ = O.square_sort(k, v, cutoff=4)
        ek, ev = CF.stable_pairs_sort(k, v)
        assert (d == ek).all() and (dv == ev).all()


def test_square_sort_degenerate_terminates():
    for n in (5, 17, 100, 1000):
        x = np.full(n, 7, np.uint64)
        d, _, st = O.square_sort(x, cutoff=4)
        assert (d == 7).all()
        assert st.degenerate >= 1 and st.single_value_buckets >= 1
    x = np.array([3] * 500 + [9] * 3, np.uint64)
    d, _, st = O.square_sort(x, cutoff=4)
    assert (d == np.sort(x)).all()


def test_square_sort_seed_and_source_invariance():
    rng = np.random.default_rng(12)
    x = rng.integers(0, 1000, 20000, dtype=np.uint64)
    ref = None
    for seed in (0, 1, 2):
        for src in (False, True):
            d, _, _ = O.square_sort(x, seed=seed, sample_from_input=src)
            ref = d if ref is None else ref
            assert (d == ref).all()


def test_level_matches_closed_form():
    rng = np.random.default_rng(14)
    for n, card in ((1000, 2**32), (4096, 2**32), (2000, 30), (999, 3)):
        x = rng.integers(0, card, n, dtype=np.uint64)
        post, _, P, be, r, deg = O.level(x, seed=3)
        m, c, e = O.column_layout(n)
        D = x.copy()
        for a, b in zip(c, e):
            D[a:b] = np.sort(D[a:b])
        dc, _, bc = CF.skew_transpose(D, P)
        assert (post == dc).all() and (be == bc).all()
        Pw, rw, dw = O.sample_pivots(O.root_key(3), x, D)
        assert (P == Pw).all() and r == rw and deg == dw


# ---------------------------------------------------------------- signed / IEEE keys (L25)
@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_total_order_ints_match_numpy(dt):
    rng = np.random.default_rng(21)
    info = np.iinfo(dt)
    x = rng.integers(info.min, info.max, 3000, dtype=dt, endpoint=True)
    x[:4] = [info.min, info.max, 0, -1]
    k = O.total_order_key(x)
    assert (O.from_total_order_key(k, dt) == x).all()
    order = np.argsort(k, kind="stable")
    assert (x[order] == np.sort(x)).all()          # unsigned order of the key = signed order
    assert k[0] == 0 and k[1] == np.iinfo(k.dtype).max  # extremes map to the extremes
    d, _ = O.square_sort_mapped(x, seed=4)
    assert (d == np.sort(x)).all()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_total_order_floats(dt):
    rng = np.random.default_rng(22)
    x = (rng.standard_normal(2000) * 10.0 ** rng.integers(-30, 30, 2000)).astype(dt)
    k = O.total_order_key(x)
    assert (O.from_total_order_key(k, dt).view(k.dtype) == x.view(k.dtype)).all()  # bijection
    d, _ = O.square_sort_mapped(x, seed=5)
    assert (d == np.sort(x)).all()                  # finite, no -0: numpy's order
    # the special values, in IEEE 754 totalOrder
    inf, u = np.inf, (np.uint32 if dt == np.float32 else np.uint64)
    w = np.dtype(u).itemsize * 8
    nan = np.array([1 << (w - 1) | ((1 << (w - 1)) - 1)], u).view(dt)[0]   # -NaN (all ones)
    pnan = np.array([(1 << (w - 1)) - 1], u).view(dt)[0]                   # +NaN
    want = np.array([nan, -inf, -np.finfo(dt).max, -1.0, -np.finfo(dt).tiny, -0.0, 0.0,
                     np.finfo(dt).tiny, 1.0, np.finfo(dt).max, inf, pnan], dt)
    perm = np.random.default_rng(3).permutation(len(want))
    got, _ = O.square_sort_mapped(want[perm], seed=1, cutoff=4)
    assert (got.view(u) == want.view(u)).all()

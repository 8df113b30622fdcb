"""Full-size parity: the CUDA path against the CPU oracle ITSELF, element by
element, at BASELINE.json's sizes (cfg4's four 2^26 variants, cfg5 = 2^28,
cfg5p = 2^27 pairs), and one level's intermediate state (pivots, accepted round,
bucket ends, post-SkewTranspose array) at cfg5-shaped sizes for u32 and u64
keys.  The oracle is single-threaded C (~100 s at 2^28); the oracle runs are
started together on a thread pool (ctypes releases the GIL), so the module
costs about as long as the slowest one."""
import concurrent.futures as cf

import numpy as np
import pytest

import oracle as O
import sqinputs as S

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2407_14801_b200 as sq  # noqa: E402

SORTS = ["cfg4_sorted", "cfg4_reverse", "cfg4_swapped", "cfg4_nonsquare", "cfg5", "cfg5p"]
# (name, n, key dtype, cardinality): cfg5-shaped levels (m = 8192 and 16384: the 8K and
# 16K column classes) and a u64 level of cfg3's recipe at full size (degenerate pivots)
LEVELS = [("u32_2^26", 1 << 26, np.uint32, 2**32), ("u32_2^28", 1 << 28, np.uint32, 2**32),
          ("u64_2^24_dup", 1 << 24, np.uint64, 1000), ("u64_2^26", 1 << 26, np.uint64, 2**64)]


def _level_input(n, dt, card):
    rng = np.random.default_rng(n ^ 0x5eed)
    if card == 2**64:
        return rng.integers(0, 2**63, n, dtype=np.uint64) * 2 + rng.integers(0, 2, n, dtype=np.uint64)
    return rng.integers(0, card, n, dtype=np.uint64).astype(dt)


@pytest.fixture(scope="module")
def oracle_results():
    """All oracle runs of the module, in parallel threads (plain C: GIL released)."""
    def sort_job(cfg):
        keys, vals = S.config(cfg)
        d, dv, _ = O.square_sort(keys, vals, seed=S.CONFIGS[cfg][2])
        return d.astype(keys.dtype), dv

    def level_job(spec):
        _, n, dt, card = spec
        keys = _level_input(n, dt, card)
        post, _, P, be, r, deg = O.level(keys, seed=91, sample_from_input=True)
        return post, P, be, r, deg

    with cf.ThreadPoolExecutor(max_workers=len(SORTS) + len(LEVELS)) as ex:
        futs = {("sort", c): ex.submit(sort_job, c) for c in SORTS}
        futs.update({("level", s[0]): ex.submit(level_job, s) for s in LEVELS})
        return {k: f.result() for k, f in futs.items()}


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("cfg", SORTS)
def test_full_size_sort_vs_oracle(cfg, oracle_results):
    keys, vals = S.config(cfg)
    seed = S.CONFIGS[cfg][2]
    want, want_v = oracle_results[("sort", cfg)]
    k = _dev(keys)
    if vals is not None:
        v = _dev(vals)
        sq.sort_pairs_u32_u32(k, v, seed)
        assert np.array_equal(_host(v), want_v)
    else:
        sq.sort_u32(k, seed)
    assert np.array_equal(_host(k), want)


@pytest.mark.parametrize("spec", LEVELS, ids=[s[0] for s in LEVELS])
def test_full_size_level_vs_oracle(spec, oracle_results):
    name, n, dt, card = spec
    post, P, be, r, deg = oracle_results[("level", name)]
    keys = _level_input(n, dt, card)
    m = O.ceil_sqrt(n)
    tdt = torch.uint32 if dt == np.uint32 else torch.uint64
    src = _dev(keys)
    dst = torch.empty_like(src)
    piv = torch.empty(m - 1, dtype=tdt, device="cuda")
    bend = torch.empty(m, dtype=torch.uint32, device="cuda")
    info = torch.empty(2, dtype=torch.uint32, device="cuda")
    (sq.debug_level_u32 if dt == np.uint32 else sq.debug_level_u64)(src, dst, 91, piv, bend, info)
    assert to_list(info) == [r, deg]
    assert np.array_equal(_host(piv).astype(np.uint64), P)
    assert np.array_equal(_host(bend).astype(np.uint64), be)
    assert np.array_equal(_host(dst).astype(np.uint64), post)
    if card == 1000:
        assert deg == 1  # 4095 draws from 1000 values: the resample cap is hit


def to_list(t):
    return _host(t).tolist()

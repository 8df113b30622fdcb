"""Statistical checks of the GPU pivot sampler against the paper's analysis (SURVEY
8(f) f2): one SquareSort level of the GPU path (sq_debug_level_u32, the sampler and
the bucket boundaries of the sort) on distinct keys, many seeds.

* accepted sampling rounds: mean = 1/p with p = prod_{i<m-1} (n-1-i)/n for distinct
  keys (a round succeeds iff the m-1 draws hit distinct positions, none of them the
  minimum; P:635-638 bounds E[rounds] by e^2);
* Prop. p-distrupper: Pr[n_i >= t sqrt(n)] <= e^(-0.9 t + 0.1);
* Prop. p-supper: Pr[n_1 <= s] <= e^2 s / sqrt(n);
* the lemma P:697-700: E[sum n_i log n_i] <= n log n / 2 + 4 e n.
Every empirical frequency is compared with its bound plus four binomial standard
errors (the bounds are loose; a wrong sampler -- e.g. one that draws from a
fixed sub-range or repeats a round -- violates them)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2407_14801_b200 as sq  # noqa: E402

N = 1 << 16
M = 256
SEEDS = 300


@pytest.fixture(scope="module")
def levels():
    rng = np.random.default_rng(2407)
    keys = rng.permutation(N).astype(np.uint32)  # distinct keys: value = rank
    src = torch.from_numpy(keys).cuda()
    dst = torch.empty_like(src)
    piv = torch.empty(M - 1, dtype=torch.uint32, device="cuda")
    bend = torch.empty(M, dtype=torch.uint32, device="cuda")
    info = torch.empty(2, dtype=torch.uint32, device="cuda")
    rounds, sizes = [], []
    for s in range(SEEDS):
        sq.debug_level_u32(src, dst, 10_000 + s, piv, bend, info)
        torch.cuda.synchronize()
        r, deg = info.cpu().tolist()
        assert deg == 0
        e = bend.cpu().numpy().astype(np.int64)
        sizes.append(np.diff(np.concatenate([[0], e])))
        rounds.append(r + 1)
    return np.array(rounds, float), np.array(sizes)


def test_bucket_sizes_partition_the_level(levels):
    _, sizes = levels
    assert (sizes.sum(axis=1) == N).all() and (sizes >= 1).all()  # distinct pivots: no empty bucket


def test_mean_rounds(levels):
    rounds, _ = levels
    p = np.prod([(N - 1 - i) / N for i in range(M - 1)])
    mu, sd = 1 / p, math.sqrt(1 - p) / p
    assert abs(rounds.mean() - mu) < 4 * sd / math.sqrt(len(rounds))
    assert rounds.mean() <= math.e ** 2


@pytest.mark.parametrize("t", [1, 2, 3, 4])
def test_upper_tail_prop_distrupper(levels, t):
    _, sizes = levels
    frac = (sizes >= t * math.sqrt(N)).mean()
    bound = math.exp(-0.9 * t + 0.1)
    cnt = sizes.size
    assert frac <= bound + 4 * math.sqrt(bound * (1 - bound) / cnt)
    # and the tail is not degenerate: exponential-like spacings put ~e^-t of the buckets there
    assert frac >= 0.25 * math.exp(-t)


@pytest.mark.parametrize("s", [2, 8, 32])
def test_lower_tail_prop_supper(levels, s):
    _, sizes = levels
    frac = (sizes[:, 0] <= s).mean()
    bound = math.e ** 2 * s / math.sqrt(N)
    assert frac <= bound + 4 * math.sqrt(min(bound, 1) / len(sizes))


def test_expected_n_log_n(levels):
    _, sizes = levels
    val = (sizes * np.log2(sizes)).sum(axis=1).mean()
    assert val <= 0.5 * N * math.log2(N) + 4 * math.e * N

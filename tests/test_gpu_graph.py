"""GPU: repeated small sorts replayed as one CUDA graph per level (engine.cuh
GraphCache).  The first call with given (buffer, n, seed) runs the ordinary path
and records the level's needs, the second captures the level, later calls replay
it -- every call must still sort the buffer's CURRENT contents bit-exactly
(integer work, bit-exact)."""
import numpy as np
import pytest

import oracle as O
import sqinputs as S
from tests import closed_forms as CF

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2407_14801_b200 as sq  # noqa: E402


def _fill(t, a):
    t.copy_(torch.from_numpy(np.ascontiguousarray(a)))


@pytest.mark.parametrize("n", [(1 << 16), (1 << 20), (1 << 20) + 12345, 40000])
def test_replayed_u32_fresh_data_every_call(n):
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for call in range(5):
        keys = S.uniform_u32(n, 100 + call)
        _fill(buf, keys)
        sq.sort_u32(buf, 1)
        assert np.array_equal(buf.cpu().numpy(), np.sort(keys)), call
        st = sq.get_stats()
        assert st["levels"] == 1 and st["kernel_launches"] > 0 and st["host_syncs"] >= 1, st


def test_replayed_vs_oracle_and_seeds():
    n = 1 << 16
    keys = S.uniform_u32(n, 1)
    want, _, _ = O.square_sort(keys, seed=1)
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for seed in (1, 2, 1, 2, 3, 1):  # entries per seed, replays interleaved
        _fill(buf, keys)
        sq.sort_u32(buf, seed)
        assert np.array_equal(buf.cpu().numpy().astype(np.uint64), want), seed


def test_replayed_two_buffers_and_trim():
    n = 1 << 18
    a = torch.empty(n, dtype=torch.uint32, device="cuda")
    b = torch.empty(n, dtype=torch.uint32, device="cuda")
    for call in range(4):
        ka, kb = S.uniform_u32(n, 7 + call), S.uniform_u32(n, 50 + call) % 1000
        _fill(a, ka)
        _fill(b, kb)
        sq.sort_u32(a, 5)
        sq.sort_u32(b, 5)
        assert np.array_equal(a.cpu().numpy(), np.sort(ka))
        assert np.array_equal(b.cpu().numpy(), np.sort(kb))
        if call == 2:
            sq.trim_memory()  # drops the cached graphs; the next calls start over


def test_replayed_pairs_stable_and_u64():
    n = 1 << 18
    rng = np.random.default_rng(3)
    k = torch.empty(n, dtype=torch.uint32, device="cuda")
    v = torch.empty(n, dtype=torch.uint32, device="cuda")
    k64 = torch.empty(n, dtype=torch.uint64, device="cuda")
    for call in range(4):
        keys = rng.integers(0, 5000, n, dtype=np.uint64).astype(np.uint32)
        vals = np.arange(n, dtype=np.uint32)
        _fill(k, keys)
        _fill(v, vals)
        sq.sort_pairs_u32_u32(k, v, 2)
        ek, ev = CF.stable_pairs_sort(keys, vals)
        assert np.array_equal(k.cpu().numpy(), ek) and np.array_equal(v.cpu().numpy(), ev), call
        x = rng.integers(0, 2**64, n, dtype=np.uint64)
        _fill(k64, x)
        sq.sort_u64(k64, 4)
        assert np.array_equal(k64.cpu().numpy(), np.sort(x)), call


def test_replayed_on_side_stream():
    n = 1 << 17
    s = torch.cuda.Stream()
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for call in range(4):
        keys = S.uniform_u32(n, 300 + call)
        _fill(buf, keys)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            sq.sort_u32(buf, 1, stream=s)
        s.synchronize()
        assert np.array_equal(buf.cpu().numpy(), np.sort(keys)), call

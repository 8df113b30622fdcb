"""GPU: the library's environment knobs that switch code paths read at load time
(SQ_SAMPLE_SPLIT: the multi-CTA candidate gather of the sampler, k_sample_gather;
SQ_SMALL_CLASSES: the latency shapes and class set of small levels).  The default
process exercises one setting of each at a given size; here every setting runs the
same checks in a fresh process: one level against the oracle's level (pivots,
accepted round, bucket ends, the post-SkewTranspose array), a
forced-tile multi-level sort with several segments per level, and replayed small
sorts -- all bit-exact."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch
import oracle as O, sqinputs as S
import paper_2407_14801_b200 as sq

def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()

# one level vs the oracle's level (sampling from the level input, L9)
for n, card in [(1 << 16, 2**32), (1 << 20, 2**32), (100003, 2**32), (50000, 7), (1 << 22, 2**32)]:
    rng = np.random.default_rng(n ^ card)
    keys = rng.integers(0, card, n, dtype=np.uint64).astype(np.uint32)
    post, _, P, be, r, deg = O.level(keys, seed=77, sample_from_input=True)
    m = O.ceil_sqrt(n)
    src = dev(keys); dst = torch.empty_like(src)
    piv = torch.empty(m - 1, dtype=torch.uint32, device="cuda")
    bend = torch.empty(m, dtype=torch.uint32, device="cuda")
    info = torch.empty(2, dtype=torch.uint32, device="cuda")
    sq.debug_level_u32(src, dst, 77, piv, bend, info)
    assert np.array_equal(piv.cpu().numpy().astype(np.uint64), P), ("pivots", n, card)
    assert np.array_equal(bend.cpu().numpy().astype(np.uint64), be), ("bucket ends", n, card)
    assert info.cpu().numpy().tolist() == [r, deg], ("round", n, card)
    assert np.array_equal(dst.cpu().numpy().astype(np.uint64), post), ("transposed", n, card)

# forced small tile: columns and buckets beyond one CTA recurse, many segments per level
# (the sampler runs per segment)
for tile in (256, 1024):
    sq.set_max_tile(tile)
    for n in (1 << 17, (1 << 18) + 777):
        keys = S.uniform_u32(n, n & 0xff)
        t = dev(keys); sq.sort_u32(t, 3)
        assert np.array_equal(t.cpu().numpy(), np.sort(keys)), ("forced tile", tile, n)
    k, v = S.generate("perm_pairs_u32", 1 << 16, 5)
    tk, tv = dev(k), dev(v); sq.sort_pairs_u32_u32(tk, tv, 5)
    o = np.argsort(k, kind="stable")
    assert np.array_equal(tk.cpu().numpy(), k[o]) and np.array_equal(tv.cpu().numpy(), v[o])
sq.set_max_tile(0)

# u64 with duplicates and replayed small sorts (graph path), fresh data every call
k64, _ = S.generate("dup1000_u64", 1 << 18, 3)
t = dev(k64); sq.sort_u64(t, 9)
assert np.array_equal(t.cpu().numpy(), np.sort(k64))
for n in (1 << 16, 1 << 18, (1 << 20) + 12345):
    buf = torch.empty(n, dtype=torch.uint32, device="cuda")
    for call in range(4):
        keys = S.uniform_u32(n, 40 + call)
        buf.copy_(torch.from_numpy(keys)); sq.sort_u32(buf, 1)
        assert np.array_equal(buf.cpu().numpy(), np.sort(keys)), ("replay", n, call)
print("knobs ok")
"""


@pytest.mark.parametrize("env", [
    {"SQ_SAMPLE_SPLIT": "1"},                 # every sample gathered by k_sample_gather
    {"SQ_SAMPLE_SPLIT": "1000000000"},        # none
    {"SQ_SMALL_CLASSES": "0"},                # small levels with the throughput shapes and all classes
    {"SQ_SAMPLE_SPLIT": "1", "SQ_SMALL_CLASSES": "0", "SQ_CONCURRENT_CLASSES": "0"},
])
def test_paths_selected_by_environment(env):
    e = dict(os.environ)
    e.update(env)
    e["PYTHONPATH"] = ROOT + os.pathsep + e.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "knobs ok" in r.stdout, (env, r.stdout[-2000:], r.stderr[-4000:])

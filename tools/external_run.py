"""Out-of-core SquareSort at scale (f4): 2^k uint64 keys in a memory-mapped file (the
paper's external-sort workload), sorted into a second mapped file with a
device budget of 2^b keys; prints wall time, ns per key and the level statistics.
  python tools/external_run.py [log2 n] [log2 budget] [dir]"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_14801_b200 import external as E  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
lb = int(sys.argv[2]) if len(sys.argv) > 2 else 27
d = sys.argv[3] if len(sys.argv) > 3 else tempfile.mkdtemp()
n = 1 << lg
src = np.memmap(os.path.join(d, "keys.bin"), dtype=np.uint64, mode="w+", shape=(n,))
dst = np.memmap(os.path.join(d, "out.bin"), dtype=np.uint64, mode="w+", shape=(n,))
rng = np.random.default_rng(lg)
step = 1 << 24
for i in range(0, n, step):
    src[i:i + step] = rng.integers(0, 2**64 - 1, min(step, n - i), dtype=np.uint64, endpoint=True)
st = {}
t0 = time.perf_counter()
E.sort_external(src, dst, seed=1, budget_keys=1 << lb, stats=st)
dt = time.perf_counter() - t0
ok = all(bool(np.all(dst[i:i + step + 1][1:] >= dst[i:i + step + 1][:-1])) for i in range(0, n, step))
print(json.dumps({"n": n, "budget_keys": 1 << lb, "seconds": dt, "ns_per_key": dt * 1e9 / n, "sorted": ok,
                  "levels": st["levels"], "groups": st["groups"], "round": st["round"]}), flush=True)
for f in ("keys.bin", "out.bin"):
    os.unlink(os.path.join(d, f))

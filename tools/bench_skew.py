"""Standalone sq_skew_transpose / _u64 timing (the north star's fourth call):
cfg2's 1024 x 1024 check and 8192 x 8192 (2^26 keys), u32 and u64, columns
sorted, pivots = every m-th key of the sorted input (distinct), cursors computed
on the device.  Prints ms per call (CUDA events, median of 10 after 3 warm-ups)
and the achieved fraction of the measured HBM copy peak on the algorithmic
bytes 2*w*n (one read, one write)."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_14801_b200 as sq  # noqa: E402

try:
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    HBM = 6650.0
out = []
for m, dt in ((1024, torch.uint32), (8192, torch.uint32), (8192, torch.uint64)):
    n = m * m
    g = torch.Generator(device="cuda").manual_seed(m)
    hi = 2**32 if dt == torch.uint32 else 2**62
    x = torch.randint(0, hi, (n,), device="cuda", generator=g, dtype=torch.int64)
    x = x.view(m, m).sort(dim=1).values.reshape(-1).to(dt)  # row r = column r of the matrix
    piv = x.to(torch.int64).sort().values[m::m][: m - 1].to(dt).contiguous()
    dst = torch.empty_like(x)
    bo = torch.empty(m, dtype=torch.uint32, device="cuda")
    for _ in range(3):
        sq.skew_transpose(x, dst, m, m, piv, buc_out=bo)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sq.skew_transpose(x, dst, m, m, piv, buc_out=bo)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    sq.profile(True)
    sq.profile_read()
    sq.skew_transpose(x, dst, m, m, piv, buc_out=bo)
    torch.cuda.synchronize()
    sq.profile(False)
    roles = {k: round(v[1], 4) for k, v in sq.profile_read().items()}
    w = x.element_size()
    gbs = 2 * w * n / (ms / 1e3) / 1e9
    ok = int(bo[-1].item()) == n
    out.append({"m": m, "dtype": str(dt), "n": n, "ms": ms, "alg_gbs": gbs, "frac_of_measured": gbs / HBM,
                "buc_out_last_ok": ok, "host_syncs": sq.get_stats()["host_syncs"], "roles_ms": roles})
    print(json.dumps(out[-1]), flush=True)

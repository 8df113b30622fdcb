"""The GPU analog of the paper's cutoff sweep: the on-chip capacity
(sq_set_max_tile: the largest segment one CTA sorts) from 1K to 32K keys, at
n = 2^24, 2^26, 2^28 uniform u32 keys.  Smaller capacities add SquareSort levels
(columns and buckets that do not fit recurse); prints ms per sort (median of 5
after 2 warm-ups), ns per key, levels and host syncs, one JSON line per point."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_14801_b200 as sq  # noqa: E402

for lg in (24, 26, 28):
    n = 1 << lg
    g = torch.Generator(device="cuda").manual_seed(lg)
    src = torch.randint(0, 2**32, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.uint32)
    work = torch.empty_like(src)
    for cap in (1024, 2048, 4096, 8192, 16384, 32768):
        sq.set_max_tile(cap)
        ts = []
        for it in range(7):
            work.copy_(src)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sq.sort_u32(work, lg)
            b.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b))
        st = sq.get_stats()
        ok = bool((work[1:].to(torch.int64) >= work[:-1].to(torch.int64)).all().item())
        ms = statistics.median(ts)
        print(json.dumps({"log2n": lg, "max_tile": cap, "ms": round(ms, 4), "ns_per_key": round(ms * 1e6 / n, 4),
                          "gkeys_s": round(n / ms / 1e6, 2), "levels": st["levels"],
                          "host_syncs": st["host_syncs"], "sorted": ok}), flush=True)
    sq.set_max_tile(0)

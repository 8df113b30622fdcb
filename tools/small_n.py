"""Latency of small sorts (cfg1 2^16, cfg2 2^20): median ms per sq_sort_u32 call
(CUDA events around each call, input restored outside), host-phase trace of one call."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs

for lg in (16, 18, 20):
    n = 1 << lg
    src = torch.from_numpy(sqinputs.uniform_u32(n, 1)).cuda()
    w = src.clone()
    ts = []
    for i in range(60):
        w.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sq.sort_u32(w, 1); e1.record(); torch.cuda.synchronize()
        if i >= 10: ts.append(e0.elapsed_time(e1))
    ok = bool(torch.equal(w.long(), torch.sort(src.long()).values))
    sq.profile(True); sq.profile_read(); w.copy_(src); sq.sort_u32(w, 1); torch.cuda.synchronize(); sq.profile(False)
    prof = {k: [v[0], round(v[1], 4)] for k, v in sq.profile_read().items()}
    print(json.dumps({"n": n, "ok": ok, "median_ms": round(statistics.median(ts), 4), "min_ms": round(min(ts), 4),
                      "stats": sq.get_stats(), "kernels": prof}))

import os, sys, time, json
sys.path.insert(0, "/root/repo")
import torch
import paper_2407_14801_b200 as sq
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
g = torch.Generator(device="cuda").manual_seed(1)
src = torch.randint(0, 2**32, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.uint32)
for cap in (1024, 16384):
    sq.set_max_tile(cap)
    w = src.clone(); sq.sort_u32(w, 1); torch.cuda.synchronize()
    sq.profile(True); sq.profile_read()
    w = src.clone()
    t0 = time.perf_counter(); sq.sort_u32(w, 1); torch.cuda.synchronize(); t1 = time.perf_counter()
    sq.profile(False)
    print(cap, "wall ms", round((t1 - t0) * 1e3, 2), sq.get_stats(), json.dumps({k: [v[0], round(v[1], 3)] for k, v in sq.profile_read().items()}))

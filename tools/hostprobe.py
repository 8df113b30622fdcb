import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S
kind, n, seed = S.CONFIGS["cfg5"]
k, _ = S.generate(kind, n, seed)
src = torch.from_numpy(k).cuda(); w = torch.empty_like(src)
for _ in range(3):
    w.copy_(src); sq.sort_u32(w, seed)
torch.cuda.synchronize()
# host wall time per call vs device events
for _ in range(3):
    w.copy_(src); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(); sq.sort_u32(w, seed); b.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("events ms", round(a.elapsed_time(b), 3), "host call ms", round((t1 - t0) * 1e3, 3), "total", round((t2 - t0) * 1e3, 3))
# now with a busy GPU queue ahead (host planning overlapped)
sq.profile(True); sq.profile_read()
for _ in range(3):
    w.copy_(src)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); sq.sort_u32(w, seed); b.record(); torch.cuda.synchronize()
    p = sq.profile_read()
    print("events ms", round(a.elapsed_time(b), 3), "kernel sum", round(sum(v[1] for v in p.values()), 3))

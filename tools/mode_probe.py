"""Time sq_sort_u32 on cfg5 under each big-bucket mode (exploration helper, not a bench)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S
kind, n, seed = S.CONFIGS["cfg5"]
k, _ = S.generate(kind, n, seed)
src = torch.from_numpy(k).cuda(); w = torch.empty_like(src)
for mode in [int(x) for x in sys.argv[1:]] or [1, 2, 0]:
    sq.set_big_bucket_mode(mode)
    for _ in range(2):
        w.copy_(src); sq.sort_u32(w, seed)
    torch.cuda.synchronize()
    sq.profile(True); sq.profile_read()
    ts = []
    for _ in range(5):
        w.copy_(src)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); sq.sort_u32(w, seed); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    p = sq.profile_read(); sq.profile(False)
    ok = bool((w[1:].to(torch.int64) >= w[:-1].to(torch.int64)).all())
    print("mode", mode, "ms", round(sorted(ts)[2], 3), {r: round(v[1] / 5, 3) for r, v in sorted(p.items(), key=lambda kv: -kv[1][1])}, "sorted", ok, sq.get_stats())

"""One warm-up + `--reps` SquareSort calls on a BASELINE config, for ncu runs.
(Not a bench: numbers printed under a profiler are never bench values.)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_14801_b200 as sq  # noqa: E402
import sqinputs as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
kind, n, seed = S.CONFIGS[a.cfg]
k, v = S.generate(kind, n, seed)
src = torch.from_numpy(k).cuda()
work = torch.empty_like(src)
vals = torch.from_numpy(v).cuda() if v is not None else None
for i in range(1 + a.reps):
    work.copy_(src)
    if vals is not None:
        vw = vals.clone()
        sq.sort_pairs_u32_u32(work, vw, seed)
    elif k.dtype.itemsize == 8:
        sq.sort_u64(work, seed)
    else:
        sq.sort_u32(work, seed)
torch.cuda.synchronize()
print("ok", sq.get_stats())

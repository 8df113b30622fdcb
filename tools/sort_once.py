"""One sq_sort_u32 of cfg5 (for ncu captures of single kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S
kind, n, seed = S.CONFIGS["cfg5"]
if len(sys.argv) > 1:  # optional: input kind (sqinputs) and log2 n
    kind, n = sys.argv[1], 1 << int(sys.argv[2]) if len(sys.argv) > 2 else n
k, _ = S.generate(kind, n, seed)
w = torch.from_numpy(k).cuda()
sq.sort_u32(w, seed)
torch.cuda.synchronize()
print("sorted", bool((w[1:].to(torch.int64) >= w[:-1].to(torch.int64)).all()))

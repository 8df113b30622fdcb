"""One sort of cfg5 (or of `kind [log2 n]`, pairs when the generator gives values),
for ncu captures of single kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S
kind, n, seed = S.CONFIGS["cfg5"]
if len(sys.argv) > 1:  # optional: input kind (sqinputs) and log2 n
    kind, n = sys.argv[1], 1 << int(sys.argv[2]) if len(sys.argv) > 2 else n
k, v = S.generate(kind, n, seed)
w = torch.from_numpy(k).cuda()
if v is not None:
    sq.sort_pairs_u32_u32(w, torch.from_numpy(v).cuda(), seed)
elif w.dtype == torch.uint64:
    sq.sort_u64(w, seed)
else:
    sq.sort_u32(w, seed)
torch.cuda.synchronize()
print("sorted", bool((w[1:].to(torch.int64) >= w[:-1].to(torch.int64)).all()))

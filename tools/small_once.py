"""Five sq_sort_u32 calls of 2^16 keys on one buffer (the 3rd onward replay the
level's CUDA graph) -- for launch lists of the small-n path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
src = torch.from_numpy(sqinputs.uniform_u32(n, 1)).cuda()
w = src.clone()
for i in range(5):
    w.copy_(src)
    sq.sort_u32(w, 1)
torch.cuda.synchronize()
print("ok", bool(torch.equal(w.long(), torch.sort(src.long()).values)))

"""One cfg5 sort (2^28 uniform u32, seed 5) in the big-bucket mode given by argv[1]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S
sq.set_big_bucket_mode(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
k = torch.from_numpy(S.uniform_u32(1 << 28, 5)).cuda()
sq.sort_u32(k, 5)
torch.cuda.synchronize()
print("ok", bool((k[1:].long() >= k[:-1].long()).all()))

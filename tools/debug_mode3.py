import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_14801_b200 as sq
import sqinputs as S
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
sq.set_big_bucket_mode(3)
keys = torch.from_numpy(S.uniform_u32(1 << lg, 5)).cuda()
w = keys.clone()
sq.sort_u32(w, 5)
torch.cuda.synchronize()
ref = torch.sort(keys.long()).values
bad = (w.long() != ref).nonzero().flatten()
print("n", 1 << lg, "mismatches", bad.numel(), "stats", sq.get_stats())
if bad.numel():
    i = int(bad[0]); j = int(bad[-1])
    print("first", i, "last", j, "span", j - i)
    print("got", w[i-3:i+5].tolist()); print("want", ref[i-3:i+5].tolist())
    # sortedness breaks
    d = (w[1:].long() < w[:-1].long()).nonzero().flatten()
    print("unsorted breaks", d.numel(), d[:10].tolist())
    # multiset equal?
    print("sum equal", int(w.long().sum()) == int(keys.long().sum()))
    # which top-level bucket holds the bad range, and its size class
    m = 16384 if lg == 28 else int(np.ceil(np.sqrt(1 << lg)))
    dst = torch.empty_like(keys); piv = torch.empty(m - 1, dtype=torch.uint32, device="cuda")
    be = torch.empty(m, dtype=torch.uint32, device="cuda"); info = torch.empty(2, dtype=torch.uint32, device="cuda")
    sq.debug_level_u32(keys, dst, 5, piv, be, info)
    torch.cuda.synchronize()
    be = be.cpu().numpy().astype(np.int64); st = np.concatenate([[0], be[:-1]])
    for pos in (i, j):
        b = int(np.searchsorted(be, pos, side="right"))
        print("pos", pos, "bucket", b, "start", st[b], "size", be[b] - st[b], "offset in bucket", pos - st[b])
    wb = int(np.searchsorted(be, int(torch.searchsorted(ref, w[i + 3].long())), side="right"))
    print("wrong keys belong to bucket", wb, "start", st[wb], "size", be[wb] - st[wb])

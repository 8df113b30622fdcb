"""One sort of uniform u32 keys at each n in argv (log2), for an ncu launch list of
DRAM bytes per kernel (the per-level IO check):
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --csv --log-file launches.csv python tools/level_bytes.py 20 22 24 26 28 30
Markers: an empty torch kernel (fill_) separates the sizes in the launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_14801_b200 as sq  # noqa: E402

marker = torch.zeros(1, device="cuda")
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    g = torch.Generator(device="cuda").manual_seed(lg)
    w = torch.randint(0, 2**32, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.uint32)
    torch.cuda.synchronize()
    marker.fill_(lg)  # separator in the launch list
    sq.sort_u32(w, lg)
    torch.cuda.synchronize()
    print(lg, sq.get_stats(), flush=True)
    del w

"""Multi-GPU SquareSort level (paper_2407_14801_b200.dist) under torchrun: every rank
holds 2^k uniform u32 keys (weak scaling), the level sorts all of them; prints the
max-over-ranks device time and checks the global order across rank boundaries.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29511 tools/dist_sort.py [log2 keys per rank]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2407_14801_b200 import dist as D  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
g = torch.Generator(device="cuda").manual_seed(1000 + rank)
block = torch.randint(0, 2**32, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.uint32)
for it in range(4):
    dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out, info = D.sort_distributed_u32(block, 7, dist)
    b.record()
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
o = out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
lo_hi = torch.tensor([int(o[0]) if o.numel() else -1, int(o[-1]) if o.numel() else -1], device="cuda")
allb = [torch.zeros_like(lo_hi) for _ in range(world)]
dist.all_gather(allb, lo_hi)
ok = bool((o[1:] >= o[:-1]).all().item()) and all(
    allb[q][1] <= allb[q + 1][0] for q in range(world - 1) if allb[q][1] >= 0 and allb[q + 1][0] >= 0)
if rank == 0:
    print(json.dumps({"ranks": world, "keys_per_rank": n, "ms_max_over_ranks": float(ms.item()),
                      "gkeys_s": world * n / float(ms.item()) / 1e6, "sorted_across_ranks": ok,
                      "round": info["round"]}), flush=True)
dist.destroy_process_group()

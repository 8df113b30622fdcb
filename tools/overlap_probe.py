"""Sort time alone vs. with a concurrent 1 GB H2D + D2H copy pair in flight."""
import time
import torch
import paper_2407_14801_b200 as sq
n = 1 << 28
h1 = torch.empty(n, dtype=torch.uint32).pin_memory()
h2 = torch.empty(n, dtype=torch.uint32).pin_memory()
d1 = torch.empty(n, dtype=torch.uint32, device="cuda")
d2 = torch.empty(n, dtype=torch.uint32, device="cuda")
keys = torch.randint(0, 2**32, (n,), dtype=torch.int64, device="cuda").to(torch.uint32)
work = torch.empty_like(keys)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()
def sort_once():
    work.copy_(keys)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    t0 = time.perf_counter()
    sq.sort_u32(work, 1)
    t1 = time.perf_counter()
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b), (t1 - t0) * 1e3
for _ in range(2): sort_once()
print("alone", [sort_once() for _ in range(3)])
for mode in ("h2d", "d2h", "both"):
    res = []
    for _ in range(3):
        torch.cuda.synchronize()
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        time.sleep(0.002)
        res.append(sort_once())
    print(mode, res)

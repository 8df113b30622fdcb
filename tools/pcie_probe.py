"""H2D / D2H copy bandwidth alone and concurrently (pinned host buffers)."""
import torch, time
n = 1 << 28
h1 = torch.empty(n, dtype=torch.uint32).pin_memory()
h2 = torch.empty(n, dtype=torch.uint32).pin_memory()
d1 = torch.empty(n, dtype=torch.uint32, device="cuda")
d2 = torch.empty(n, dtype=torch.uint32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
GB = n * 4 / 1e9
for name, f in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(f)
    print(name, round(ms, 2), "ms", round(GB / ms * 1e3, 1), "GB/s per direction")

"""The paper's experiment set on the GPU: sq_sort_u32 time
per item across n for the paper's four distributions -- a random permutation,
binary keys, uniform in {1..n} and uniform in {1..sqrt n} -- plus uniform
u32.  Prints a markdown table (Gkeys/s and ns per n*log2(n)); every output is
checked sorted with the input's sum.  Not a bench line: a characterisation."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S

KINDS = [("uniform_u32", "uniform u32"), ("perm_pairs_u32", "permutation"), ("binary_u32", "binary"),
         ("uniform_n_u32", "uniform {1..n}"), ("uniform_sqrt_u32", "uniform {1..sqrt n}")]


def time_sort(src, reps):
    w = torch.empty_like(src)
    ts = []
    for i in range(reps + 2):
        w.copy_(src)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sq.sort_u32(w, 1)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ok = bool((w[1:].to(torch.int64) >= w[:-1].to(torch.int64)).all()) and \
        int(w.to(torch.int64).sum()) == int(src.to(torch.int64).sum())
    return sorted(ts)[len(ts) // 2], ok


def main():
    logs = [int(x) for x in sys.argv[1:]] or list(range(16, 29, 2))
    rows = []
    for kind, name in KINDS:
        for lg in logs:
            n = 1 << lg
            k, _ = S.generate(kind, n, 11)
            src = torch.from_numpy(k.astype(np.uint32)).cuda()
            ms, ok = time_sort(src, 5 if lg >= 26 else 10)
            rows.append((name, lg, ms, n / ms / 1e6, ms * 1e6 / (n * math.log2(n)), ok))
            print(rows[-1], flush=True)
            del src
    out = ["| distribution | n | ms | Gkeys/s | ns per n·log2 n | checked |", "|---|---|---|---|---|---|"]
    for name, lg, ms, g, t, ok in rows:
        out.append(f"| {name} | 2^{lg} | {ms:.3f} | {g:.2f} | {t:.4f} | {'sorted+sum' if ok else 'FAILED'} |")
    print("\n".join(out))


if __name__ == "__main__":
    main()

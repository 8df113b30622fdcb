"""Time every BASELINE config (cfg1..cfg5, 4', 5p) through the sort ABI on one B200
and check each output against numpy's sort (stable sort by key for pairs).
A characterisation table, not the bench line (bench.py times cfg5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S


def timed(fn, reset, reps):
    ts = []
    for i in range(reps + 2):
        reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    rows = []
    for name, (kind, n, seed) in S.CONFIGS.items():
        k, v = S.generate(kind, n, seed)
        reps = 5 if n >= 1 << 26 else 10
        if v is not None:
            kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
            wk, wv = torch.empty_like(kd), torch.empty_like(vd)
            ms = timed(lambda: sq.sort_pairs_u32_u32(wk, wv, seed), lambda: (wk.copy_(kd), wv.copy_(vd)), reps)
            o = np.argsort(k, kind="stable")
            ok = np.array_equal(wk.cpu().numpy(), k[o]) and np.array_equal(wv.cpu().numpy(), v[o])
        else:
            dt = torch.uint64 if k.dtype == np.uint64 else torch.uint32
            kd = torch.from_numpy(k).cuda()
            wk = torch.empty_like(kd)
            f = sq.sort_u64 if dt == torch.uint64 else sq.sort_u32
            ms = timed(lambda: f(wk, seed), lambda: wk.copy_(kd), reps)
            ok = np.array_equal(wk.cpu().numpy(), np.sort(k))
        rows.append((name, kind, n, k.dtype.name, ms, n / ms / 1e6, ok))
        print(rows[-1], flush=True)
        del kd, wk
    print("| config | input | n | key | ms | Gkeys/s | = numpy |\n|---|---|---|---|---|---|---|")
    for name, kind, n, dt, ms, g, ok in rows:
        print(f"| {name} | {kind} | {n} | {dt} | {ms:.3f} | {g:.2f} | {'yes' if ok else 'NO'} |")


if __name__ == "__main__":
    main()

"""Aggregate an `ncu --page source --csv --print-source=cuda,sass` export by CUDA
source line: warp instructions executed and stall samples per (file, line)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file, hdr, agg = None, None, {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            try:
                ie = float(r[hdr.index("Instructions Executed")] or 0)
                st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except ValueError:
                continue
            agg[(cur_file, int(r[0]))] = (ie, st, r[1].strip())
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"{path}: {ti:.4g} warp instructions, {ts:.4g} stall samples")
    for (f, l), (ie, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ie / ti * 100:5.1f}% ins {st / ts * 100:5.1f}% stall  {f}:{l}  {src[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

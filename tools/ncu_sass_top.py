"""Summarise an `ncu --page source --csv --print-source=sass` export: total warp
instructions and the hottest SASS lines by executed instructions and stall samples."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if len(r) > 3 and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            try:
                float(r[hdr.index("Instructions Executed")] or 0)
            except ValueError:
                continue
            data.append(dict(zip(hdr, r)))
    return data


def main(path, top=30, key="Instructions Executed"):
    data = load(path)
    f = lambda r, k: float(r.get(k) or 0)
    tot = sum(f(r, "Instructions Executed") for r in data)
    stall = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"{path}: {len(data)} SASS lines, {tot:.4g} warp instructions, {stall:.4g} stall samples")
    idx = sorted(range(len(data)), key=lambda i: -f(data[i], key))[:top]
    for i in sorted(idx):
        r = data[i]
        print(f"{i:5d} ins {f(r,'Instructions Executed')/tot*100:5.2f}%  stall "
              f"{f(r,'Warp Stall Sampling (All Samples)')/max(stall,1)*100:5.2f}%  {r['Source'][:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30,
         sys.argv[3] if len(sys.argv) > 3 else "Instructions Executed")

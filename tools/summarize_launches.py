"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`) of one bench.py run: per kernel role, launches per sort
call, device time and DRAM bytes per launch (cold-cache, serialised -- shares, not
absolutes), written as markdown and as profiles/ncu_traffic.json (bytes per launch
by role, read by bench.py's roofline.traffic)."""
import csv
import json
import sys
from collections import OrderedDict

ROLE = [("k_tile_bucket_plan", "plan"), ("k_colsort", "colsort"), ("k_transpose", "transpose"), ("k_bucketsort", "bucketsort"),
        ("k_merge_pass", "merge"), ("k_merge_split", "merge"), ("k_pairsort", "pairsort"), ("k_clustersort", "clustersort"), ("k_sample", "sample"),
        ("k_select", "select"), ("k_segmat", "segmat"), ("k_tile", "tiles"), ("k_piece_plan", "tiles"),
        ("k_bucket_sizes", "plan"), ("k_bucket_offsets", "plan"), ("k_bucket_plan", "plan"),
        ("k_bucket_gather", "gather"), ("k_blocksort", "smallsort"), ("k_colmin", "colmin"),
        ("k_unit_plan", "plan"), ("k_xfer", "xfer"), ("k_readback", "xfer"), ("k_gather_units", "gather"),
        ("k_binsort_cluster", "bucketsort")]


def role_of(name):
    for k, r in ROLE:
        if k in name:
            return r
    return None


def main(path, out_md, out_json, calls):
    rows = list(csv.reader(open(path)))
    hdr, cur = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = cur.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d["Grid Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = OrderedDict()
    for i in sorted(cur):
        e = cur[i]
        r = role_of(e["name"])
        if r is None:
            continue
        a = agg.setdefault(r, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += e.get("gpu__time_duration.sum", 0) / 1e6
        a[2] += e.get("dram__bytes_read.sum", 0)
        a[3] += e.get("dram__bytes_write.sum", 0)
    tot_ms = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list summary ({path}, {calls} sort calls)", "",
             "| role | launches/call | ms/call | share | DRAM read MB/call | DRAM write MB/call | DRAM bytes/launch |",
             "|---|---|---|---|---|---|---|"]
    traffic, per_call = {}, {}
    for r, (n, ms, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        per_launch = (rd + wr) / n
        traffic[r] = per_launch
        per_call[r] = n / calls
        lines.append(f"| {r} | {n / calls:g} | {ms / calls:.3f} | {ms / tot_ms * 100:.1f}% | {rd / calls / 1e6:.1f} | "
                     f"{wr / calls / 1e6:.1f} | {per_launch:.4g} |")
    lines.append(f"| total | | {tot_ms / calls:.3f} | | | | |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    json.dump({"source": path, "sort_calls": calls, "bytes_per_launch": traffic, "launches_per_call": per_call},
              open(out_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 1)

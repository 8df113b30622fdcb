"""Summarise an `ncu --set full` report (one or more kernels) as a markdown table of
the metrics the roofline discussion uses: duration, DRAM bytes and throughput,
issue/IPC, pipe utilisation, occupancy, registers and the top stall reasons."""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Executed Instructions", "Achieved Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size"]


def main(rep, out):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    kern = {}
    order = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        if key not in kern:
            kern[key] = {}
            order.append(key)
        if d["Metric Name"] in KEEP:
            kern[key][d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    raws = {}
    for r in rr[2:]:
        d = dict(zip(rh, r))
        raws[d["ID"]] = d
    lines = [f"# ncu --set full summary: {rep}", ""]
    for key in order:
        kid, name = key
        lines.append(f"## {name[:110]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m in KEEP:
            if m in kern[key]:
                lines.append(f"| {m} | {kern[key][m]} |")
        d = raws.get(kid, {})
        for m in ["dram__bytes_read.sum", "dram__bytes_write.sum"]:
            if m in d:
                lines.append(f"| {m} | {d[m]} (raw units) |")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        st.sort(reverse=True)
        lines.append("| top stall reasons (share of samples) | " +
                     ", ".join(f"{k} {v / tot * 100:.0f}%" for v, k in st[:5]) + " |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

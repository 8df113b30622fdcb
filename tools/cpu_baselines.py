"""CPU context rows for BASELINE.md section 4, on the GPU box's host: the oracle
(single-threaded SquareSort, oracle/) and std::sort (tools/cpu/stdsort.cpp), each
pinned to one core with taskset, on the configs' inputs (cfg5 full for std::sort,
a 2^25 sample for the oracle).  Prints one JSON line per measurement."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import sqinputs as S  # noqa: E402

exe = os.path.join(ROOT, "tools", "cpu", "stdsort")
subprocess.check_call(["g++", "-O3", "-march=native", "-o", exe, exe + ".cpp"])
model = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")
print(json.dumps({"host_cpu": model, "nproc": os.cpu_count()}), flush=True)
for kind, n, seed in (("u32", 1 << 16, 1), ("u32", 1 << 20, 2), ("dup64", 1 << 24, 3), ("u32", 1 << 28, 5)):
    out = subprocess.check_output(["taskset", "-c", "0", exe, kind, str(n), str(seed)], text=True)
    print(json.dumps({"impl": "std::sort, 1 core", **json.loads(out)}), flush=True)
os.sched_setaffinity(0, {0})
for name, n in (("cfg1", None), ("cfg2", None), ("cfg3", None), ("cfg5", 1 << 25)):
    keys, _ = S.config(name, n=n)
    t0 = time.perf_counter()
    O.square_sort(keys, seed=S.CONFIGS[name][2])
    dt = time.perf_counter() - t0
    print(json.dumps({"impl": "oracle SquareSort, 1 core", "config": name, "n": len(keys), "seconds": dt,
                      "mkeys_s": len(keys) / dt / 1e6}), flush=True)

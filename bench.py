#!/usr/bin/env python3
"""SquareSort throughput on B200 -- BASELINE.json's metric:
"Gkeys/s for SquareSort of 2^28 uint32 keys; fraction of 8 TB/s HBM roofline".

One step = one sq_sort_u32 call (the whole hot path: column sort, pivot
sampling, bucket count, SkewTranspose, bucket sorts, oversize levels) on
config 5 (2^28 uniform uint32 keys, seed 5; BASELINE configs[4]).  The input
(1 GiB) is restored from a pristine device copy before every step, outside the
step's CUDA events; it is larger than the 126 MB L2, so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): every rank sorts its own 2^28 keys -- replicas, no
collective on the data path; value = all ranks' keys / the max
over ranks of the summed step time.  `--impl reference` times the CPU oracle
(the reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gkeys/s for SquareSort of 2^28 uint32 keys; fraction of 8 TB/s HBM roofline"
UNIT = "Gkeys/s"
CFG = "cfg5"
NOMINAL_HBM_GBS = 8000.0
W = 4  # bytes per key


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(p.get("sm_max_mhz", 1965))
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(keys, seconds_hint=True):
    """The oracle as it stands, single-threaded, on a bounded sample of the workload."""
    import oracle as O
    n = 1 << 25  # ~10 s of single-core work
    sample = keys[:n].copy()
    t0 = time.perf_counter()
    O.square_sort(sample, seed=5)
    dt = time.perf_counter() - t0
    return {"value": n / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first 2^25 keys of the cfg5 input (uniform u32, seed 5), oracle SquareSort "
                      f"cutoff 16 / threshold 4, one run, {dt:.2f} s on 1 host core",
            "host_cpu": _cpu_model(), "host_nproc": os.cpu_count()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, rank):
    if rank != 0:
        return
    import oracle as O
    import sqinputs as S
    n = 1 << 21
    kind, _, seed = S.CONFIGS[CFG]
    keys, _ = S.generate(kind, n, seed)
    for _ in range(args.warmup):
        O.square_sort(keys, seed=seed)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.square_sort(keys, seed=seed)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms / 1e3) / 1e9
    sample = (f"2^21 keys of the cfg5 recipe (uniform u32, seed 5) per step; oracle SquareSort "
              f"(oracle/squaresort_oracle.c, cutoff 16, threshold 4), single-threaded")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "cfg5 sample: 2^21 uniform uint32 keys (seed 5) on 1 host core",
                   "n": n, "parallelism": "none (CPU oracle)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": sample, "host_cpu": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def bind_to_gpu_cpus(index: int):
    """Run on the CPUs NVML reports as affine to the GPU, so the pinned host
    buffers of the e2e leg are first-touched on the GPU's NUMA node.  Best effort:
    returns the CPU list, or None when NVML or the affinity call is unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return sorted(cpus)
    except Exception:
        pass
    return None


def max_over_ranks(x: float, dist=None) -> float:
    """The job's time is the slowest rank's (device-timed on each rank)."""
    if dist is None:
        return x
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(world: int, n: int, ms_per_step: float) -> float:
    """Whole-job Gkeys/s of `world` independent replicas of an n-key sort (weak
    scaling: every rank sorts its own n keys; the step time is the max over ranks)."""
    return world * n / (ms_per_step / 1e3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch

    import paper_2407_14801_b200 as sq
    import sqinputs as S

    torch.cuda.set_device(local)
    affinity = bind_to_gpu_cpus(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    kind, n, seed = S.CONFIGS[CFG]
    keys, _ = S.generate(kind, n, seed)
    pristine = torch.from_numpy(keys).cuda()
    work = torch.empty_like(pristine)
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 0)):
        work.copy_(pristine)
        sq.sort_u32(work, seed)
    torch.cuda.synchronize()

    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    evs, launches, stats = [], 0, None
    for _ in range(args.steps):
        work.copy_(pristine)  # restore: outside the step's events
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sq.sort_u32(work, seed)
        b.record(stream)
        evs.append((a, b))
        stats = sq.get_stats()
        launches += stats["kernel_launches"]
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    # Per-kernel device times (the roofline's launch durations): the same K steps again
    # with the library's per-launch CUDA events on -- kept out of the timed steps above,
    # whose wall time they would inflate by ~2 % (extra API calls per launch).
    sq.profile(True)
    sq.profile_read()
    for _ in range(args.steps):
        work.copy_(pristine)
        sq.sort_u32(work, seed)
    torch.cuda.synchronize()
    sq.profile(False)
    prof = sq.profile_read()
    total_ms = max_over_ranks(total_ms, dist)
    ms = total_ms / args.steps
    value = replica_value(world, n, ms)

    # sanity: the last step's output is sorted and a permutation (sum check)
    w64 = work.to(torch.int64)
    ok = bool((w64[1:] >= w64[:-1]).all().item()) and \
        int(w64.sum().item()) == int(pristine.to(torch.int64).sum().item())
    del w64

    hbm, hbm_src, sm_mhz_max = peaks()
    b_alg = 6 * W * n  # column pass + SkewTranspose + bucket pass, read + write
    # Roofline of the dominant role: every pass of the level is bound by
    # HBM bandwidth in the model -- its algorithmic bytes are one read and one write of
    # the n keys (2*w*n) -- so `achieved` = 2*w*n / the role's device time per step and
    # `frac` = achieved / the measured copy bandwidth.  The bucket phase is timed as one
    # span (its size classes and the merge passes of big buckets run concurrently on
    # side streams); its ncu traffic includes the merge passes.  The on-chip sorts'
    # ALU view (comparisons/s) is kept beside it.
    m = int(math.isqrt(n - 1)) + 1
    comps = n * math.log2(m)
    alu_peak = 148 * 64 * sm_mhz_max * 1e6 / 2 / 1e12  # T comparisons/s
    role_bytes = {"colsort": 2 * W * n, "transpose": 2 * W * n, "bucketsort": 2 * W * n,
                  "smallsort": 2 * W * n, "count": W * n}
    per_step = {k: (v[0] / args.steps, v[1] / args.steps) for k, v in prof.items()}  # role -> (launches, ms)
    cand = {k: v for k, v in per_step.items() if k in role_bytes}
    dname, (dlaunch, dms) = max(cand.items(), key=lambda kv: kv[1][1]) if cand else ("none", (1.0, 0.0))
    traffic_step = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            bpl, lpc = tj["bytes_per_launch"], tj.get("launches_per_call", {})
            parts = [dname] + (["merge"] if dname == "bucketsort" else [])
            traffic_step = sum(bpl[r] * lpc.get(r, 1) for r in parts if r in bpl) or None
        except Exception:
            traffic_step = None
    sec = dms / 1e3
    achieved = role_bytes.get(dname, 0) / sec / 1e9 if sec else 0.0
    roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic_step, "peak_source": hbm_src,
                "algorithmic_bytes_per_launch": role_bytes.get(dname, 0),
                "launch": "one timed unit per step (the bucket phase: one fork-to-join span)",
                "launches_per_step": 1, "share_of_step": dms / ms if ms > 0 else None,
                "traffic_note": "ncu dram__bytes_read+write summed over the role's kernels per sort call "
                                "(profiles/ncu_traffic.json; bucket phase incl. merge passes)",
                "alu_view": {"work": "n*log2(m) comparisons", "achieved_tcomp_s": comps / sec / 1e12 if sec else 0.0,
                             "peak_tcomp_s": alu_peak,
                             "frac": (comps / sec / 1e12) / alu_peak if sec else 0.0,
                             "peak_source": f"derived: 148 SMs x 64 ALU lanes/clk x {sm_mhz_max:.0f} MHz / 2"}}
    roles = {k: {"ms": v[1], "hbm_frac": role_bytes[k] / (v[1] / 1e3) / 1e9 / hbm}
             for k, v in per_step.items() if k in role_bytes and v[1] > 0}
    step_gbs = b_alg / (ms / 1e3) / 1e9

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "cfg5: 2^28 uniform uint32 keys, seed 5 (BASELINE configs[4])",
                   "n": n, "seed": seed, "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "inputs (1 GiB) exceed the 126 MB L2; no flush needed",
                   "restore": "D2D copy of the pristine input before each step, outside the events"},
        "hbm_roofline_step": {"b_alg_bytes": b_alg, "achieved_gbs": step_gbs,
                              "frac_of_8TBs": step_gbs / NOMINAL_HBM_GBS, "frac_of_measured": step_gbs / hbm},
        "roofline": roofline,
        "roles_hbm_frac_of_measured": roles,
        "ms_per_step_median": statistics.median(step_ms), "ms_per_step_min": min(step_ms),
        "kernels_ms_per_step": {k: v[1] / args.steps for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
        "kernel_timing": "library per-launch CUDA events (on the sort's stream) over a second pass of the same K steps "
                         "run right after the timed steps (events inside the timed steps would add ~2 % of API overhead)",
        "gpu_launches": launches,
        "clocks": clk,
        "sort_stats": stats,
        "output_check": "sorted+sum" if ok else "FAILED",
    }
    if not args.no_e2e:
        # End to end through the public host API: every step copies its n keys
        # in from pinned host memory and its n sorted keys back out.  The
        # batch call pipelines consecutive steps (copy-in of step i+1 and
        # copy-out of step i-1 overlap the sort of step i on two copy streams).
        hin = torch.empty(n, dtype=torch.uint32).pin_memory().numpy()
        np.copyto(hin, keys)
        houts = [torch.empty(n, dtype=torch.uint32).pin_memory().numpy() for _ in range(2)]
        esteps = 20
        sq.sort_u32_host_batch([hin], [houts[0]], seed)  # warm-up
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        sq.sort_u32_host_batch([hin] * esteps, [houts[i % 2] for i in range(esteps)], seed)
        b.record(stream)
        torch.cuda.synchronize()
        em = a.elapsed_time(b) / esteps
        e_ok = bool(np.all(houts[0][1:] >= houts[0][:-1]) and np.all(houts[1][1:] >= houts[1][:-1]))
        # the same step one call at a time (no overlap between steps), for context
        hs = torch.empty(n, dtype=torch.uint32).pin_memory().numpy()
        s_ms = []
        for i in range(3):
            np.copyto(hs, keys)  # restore (untimed)
            a.record(stream)
            sq.sort_u32_host(hs, seed)
            b.record(stream)
            torch.cuda.synchronize()
            if i > 0:
                s_ms.append(a.elapsed_time(b))
        sm = sum(s_ms) / len(s_ms)
        out["e2e"] = {"value": world * n / (em / 1e3) / 1e9, "unit": UNIT, "ms_per_step": em,
                      "steps": esteps, "h2d_bytes_per_step": n * W, "d2h_bytes_per_step": n * W,
                      "api": "sq_sort_u32_host_batch (pinned host buffers; every step = H2D of n keys + sort + "
                             "D2H of n keys, consecutive steps pipelined on copy streams)",
                      "output_check": "sorted" if e_ok else "FAILED",
                      "host_cpus": "GPU-affine (NVML): %s" % (f"{affinity[0]}-{affinity[-1]}" if affinity else "not set"),
                      "unpipelined": {"value": world * n / (sm / 1e3) / 1e9, "ms_per_step": sm,
                                      "api": "sq_sort_u32_host, one call per step"}}
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(keys)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

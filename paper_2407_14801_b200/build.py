"""Build libsquaresort.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

The engine is instantiated once per key type in its own translation unit
(csrc/inst_*.cu); the units compile in parallel and link into one shared
library whose exported symbols are the C ABI of include/squaresort.h.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsquaresort.so")
SOURCES = ["api.cu", "inst_u32.cu", "inst_u32m.cu", "inst_u64.cu", "inst_u64b.cu", "inst_pairs.cu", "inst_pairsb.cu",
           "inst_pairs64.cu"]
HEADERS = ["engine.cuh", "common.cuh", "blocksort.cuh", "binsort.cuh", "binclust.cuh", "level.cuh", "level2.cuh", "skew.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC"] + os.environ.get("SQ_NVCC_EXTRA", "").split()


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _hdr_time() -> float:
    hdr = os.path.join(os.path.dirname(HERE), "include", "squaresort.h")
    return max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] + [_mtime(hdr), _mtime(__file__)])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = _mtime(LIB)
    return _hdr_time() > t or any(_mtime(os.path.join(CSRC, s)) > t for s in SOURCES)


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or stale()):
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = _hdr_time()
    procs, objs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s.replace(".cu", ".o"))
        objs.append(obj)
        if not force and _mtime(obj) > max(hdr_t, _mtime(src)):
            continue
        cmd = [nvcc, *NVCC_FLAGS, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd, cwd=CSRC)))
    failed = [cmd for cmd, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    link = [nvcc, *ARCH, "-shared", "-o", LIB, *objs]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link, cwd=CSRC)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)

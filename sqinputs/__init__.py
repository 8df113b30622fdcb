"""Seeded synthetic inputs for SquareSort.

One module serves the oracle side (tests) and the GPU side (tests, bench) with
identical inputs; it holds none of the method's arithmetic.  The recipes are
BASELINE.json's five configs; the paper measures only
synthetic data, so no public dataset is stood in for.

Kinds:
  uniform_u32      key_i = x_i >> 32                      (cfg 1, 2, 4', 5)
  dup1000_u64      key_i = floor(x_i * 1000 / 2^64)       (cfg 3; P:848's low-cardinality workload)
  sorted_u32       sort(uniform_u32)                      (cfg 4)
  reverse_u32      reversed(sorted_u32)                   (cfg 4)
  swapped_u32      sorted_u32 + floor(n/200) random transpositions from the continued stream (cfg 4)
  perm_pairs_u32   keys = Fisher-Yates permutation of 0..n-1, vals_i = i (cfg 5p)
  binary_u32, uniform_n_u32, uniform_sqrt_u32  -- the paper's other distributions
where x_i is the i-th SplitMix64 output for the config seed.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsqinputs.so")
_lib = None

# name -> (kind, n, seed); BASELINE.json "configs"
CONFIGS = {
    "cfg1": ("uniform_u32", 1 << 16, 1),
    "cfg2": ("uniform_u32", 1 << 20, 2),
    "cfg3": ("dup1000_u64", 1 << 24, 3),
    "cfg4_sorted": ("sorted_u32", 1 << 26, 4),
    "cfg4_reverse": ("reverse_u32", 1 << 26, 4),
    "cfg4_swapped": ("swapped_u32", 1 << 26, 4),
    "cfg4_nonsquare": ("uniform_u32", (1 << 26) - 12345, 4),
    "cfg5": ("uniform_u32", 1 << 28, 5),
    "cfg5p": ("perm_pairs_u32", 1 << 27, 5),
}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        c64, vp = ctypes.c_uint64, ctypes.c_void_p
        L.sqg_stream.argtypes = [c64, c64, c64, vp]
        L.sqg_uniform_u32.argtypes = [c64, c64, vp]
        L.sqg_uniform_mod_u64.argtypes = [c64, c64, c64, vp]
        L.sqg_swaps_u32.argtypes = [vp, c64, c64, c64, c64]
        L.sqg_permutation_u32.argtypes = [c64, c64, vp]
        for f in ("sqg_stream", "sqg_uniform_u32", "sqg_uniform_mod_u64", "sqg_swaps_u32",
                  "sqg_permutation_u32"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().sqg_stream(seed, start, n, out.ctypes.data)
    return out


def uniform_u32(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    lib().sqg_uniform_u32(seed, n, out.ctypes.data)
    return out


def uniform_mod_u64(n: int, seed: int, card: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().sqg_uniform_mod_u64(seed, n, card, out.ctypes.data)
    return out


def generate(kind: str, n: int, seed: int):
    """Returns (keys, vals_or_None)."""
    if kind == "uniform_u32":
        return uniform_u32(n, seed), None
    if kind == "dup1000_u64":
        return uniform_mod_u64(n, seed, 1000), None
    if kind in ("sorted_u32", "reverse_u32", "swapped_u32"):
        a = np.sort(uniform_u32(n, seed))
        if kind == "reverse_u32":
            a = np.ascontiguousarray(a[::-1])
        elif kind == "swapped_u32":
            lib().sqg_swaps_u32(a.ctypes.data, n, seed, n, n // 200)
        return a, None
    if kind == "perm_pairs_u32":
        k = np.empty(n, np.uint32)
        lib().sqg_permutation_u32(seed, n, k.ctypes.data)
        return k, np.arange(n, dtype=np.uint32)
    if kind == "binary_u32":
        return (uniform_u32(n, seed) >> 31).astype(np.uint32), None
    if kind == "uniform_n_u32":
        return (1 + uniform_mod_u64(n, seed, n)).astype(np.uint32), None
    if kind == "uniform_sqrt_u32":
        return (1 + uniform_mod_u64(n, seed, max(1, math.isqrt(n)))).astype(np.uint32), None
    raise ValueError(kind)


def config(name: str, n: int | None = None):
    """Config `name` at its BASELINE size, or the same recipe at size n."""
    kind, n0, seed = CONFIGS[name]
    return generate(kind, n0 if n is None else n, seed)

"""CPU oracle for SquareSort (arXiv 2407.14801) -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper around ``oracle/squaresort_oracle.c``, a plain single-threaded
C11 implementation of the paper's Algorithms 1-3 (PAPER.md P:251-295,
P:403-451).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module; the
product package ``paper_2407_14801_b200`` never does, and the two share no
code.

Arrays are numpy: keys as ``uint64`` (u32 keys are widened -- same order),
optional payload as ``uint32``.  All indices are 0-based.
See the C file's header for citations and pin status.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "squaresort_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

u64p = ctypes.POINTER(ctypes.c_uint64)
u32p = ctypes.POINTER(ctypes.c_uint32)


class _Params(ctypes.Structure):
    _fields_ = [("cutoff", ctypes.c_uint32), ("naive_threshold", ctypes.c_uint32),
                ("resample_cap", ctypes.c_uint32), ("sample_from_input", ctypes.c_uint32)]


class _Stats(ctypes.Structure):
    _fields_ = [("nodes", ctypes.c_uint64), ("rounds", ctypes.c_uint64),
                ("degenerate", ctypes.c_uint64), ("max_depth", ctypes.c_uint64),
                ("single_value_buckets", ctypes.c_uint64)]


@dataclass
class Stats:
    nodes: int
    rounds: int
    degenerate: int
    max_depth: int
    single_value_buckets: int


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", _LIB,
                               _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.sqo_mix.restype = ctypes.c_uint64
        L.sqo_mix.argtypes = [ctypes.c_uint64]
        L.sqo_root_key.restype = ctypes.c_uint64
        L.sqo_root_key.argtypes = [ctypes.c_uint64]
        L.sqo_child_key.restype = ctypes.c_uint64
        L.sqo_child_key.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.sqo_draw.restype = ctypes.c_uint64
        L.sqo_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        L.sqo_index.restype = ctypes.c_uint64
        L.sqo_index.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.sqo_ceil_sqrt.restype = ctypes.c_uint64
        L.sqo_ceil_sqrt.argtypes = [ctypes.c_uint64]
        L.sqo_column_layout.restype = ctypes.c_uint64
        L.sqo_column_layout.argtypes = [ctypes.c_uint64, u64p, u64p]
        L.sqo_simple_sort.restype = None
        L.sqo_simple_sort.argtypes = [u64p, u32p, u64p, u32p, ctypes.c_uint64]
        L.sqo_merge_sort.restype = None
        L.sqo_merge_sort.argtypes = [u64p, ctypes.c_uint64]
        L.sqo_sample_pivots.restype = ctypes.c_uint32
        L.sqo_sample_pivots.argtypes = [ctypes.c_uint64, u64p, u64p, ctypes.c_uint64,
                                        ctypes.c_uint32, u64p, u32p]
        L.sqo_initial_bucket_cursors.restype = None
        L.sqo_initial_bucket_cursors.argtypes = [u64p, ctypes.c_uint64, u64p, u64p, u64p,
                                                 ctypes.c_uint64, ctypes.c_uint64, u64p]
        L.sqo_naive_skew_transpose.restype = None
        L.sqo_naive_skew_transpose.argtypes = [u64p, u32p, u64p, u32p, ctypes.c_uint64, u64p,
                                               u64p, ctypes.c_uint64, ctypes.c_uint64, u64p,
                                               ctypes.c_uint64, u64p]
        L.sqo_skew_transpose.restype = None
        L.sqo_skew_transpose.argtypes = [u64p, u32p, u64p, u32p, ctypes.c_uint64, u64p, u64p,
                                         ctypes.c_uint64, ctypes.c_uint64, u64p, ctypes.c_uint64,
                                         u64p, ctypes.c_uint32]
        L.sqo_square_sort.restype = ctypes.c_int
        L.sqo_square_sort.argtypes = [u64p, u32p, u64p, u32p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.POINTER(_Params), ctypes.POINTER(_Stats)]
        L.sqo_level.restype = ctypes.c_uint32
        L.sqo_level.argtypes = [u64p, u32p, u64p, u32p, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.POINTER(_Params), u64p, u64p, u32p]
        L.sqo_skew_transpose_matrix.restype = None
        L.sqo_skew_transpose_matrix.argtypes = [u64p, u32p, u64p, u32p, ctypes.c_uint64,
                                                ctypes.c_uint64, ctypes.c_uint64, u64p,
                                                ctypes.c_uint64, u64p, u64p, ctypes.c_uint32]
        _lib = L
    return _lib


def _p64(a):
    return None if a is None else a.ctypes.data_as(u64p)


def _p32(a):
    return None if a is None else a.ctypes.data_as(u32p)


def _k(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).astype(np.uint64, copy=True))


def _v(a):
    return None if a is None else np.ascontiguousarray(np.asarray(a).astype(np.uint32, copy=True))


# ---------------------------------------------------------------- RNG
def mix(x: int) -> int:
    return lib().sqo_mix(x & (2**64 - 1))


def root_key(seed: int) -> int:
    return lib().sqo_root_key(seed & (2**64 - 1))


def child_key(key: int, phase: int, idx: int) -> int:
    return lib().sqo_child_key(key, phase, idx)


def draw(key: int, r: int, i: int) -> int:
    return lib().sqo_draw(key, r, i)


def index(d: int, n: int) -> int:
    return lib().sqo_index(d, n)


# ---------------------------------------------------------------- Alg 1 pieces
def ceil_sqrt(n: int) -> int:
    return lib().sqo_ceil_sqrt(n)


def column_layout(n: int):
    """(m, col, colEnd), 0-based."""
    m = ceil_sqrt(n)
    col = np.zeros(max(m, 1), np.uint64)
    end = np.zeros(max(m, 1), np.uint64)
    lib().sqo_column_layout(n, _p64(col), _p64(end))
    return m, col[:m], end[:m]


def simple_sort(keys, vals=None):
    A, Av = _k(keys), _v(vals)
    D = np.zeros_like(A)
    Dv = None if Av is None else np.zeros_like(Av)
    lib().sqo_simple_sort(_p64(A), _p32(Av), _p64(D), _p32(Dv), len(A))
    return D if Dv is None else (D, Dv)


def merge_sort(a):
    A = _k(a)
    lib().sqo_merge_sort(_p64(A), len(A))
    return A


def sample_pivots(node: int, src, D, cap: int = 32):
    """(pivots[m-1], round, degenerate) for a level of n = len(D) items whose
    columns in D are sorted; candidates are drawn from `src`."""
    S, Dk = _k(src), _k(D)
    n = len(Dk)
    m = ceil_sqrt(n)
    P = np.zeros(max(m - 1, 1), np.uint64)
    deg = ctypes.c_uint32(0)
    r = lib().sqo_sample_pivots(node, _p64(S), _p64(Dk), n, cap, _p64(P), ctypes.byref(deg))
    return P[: m - 1], int(r), int(deg.value)


def initial_bucket_cursors(D, col, colEnd, pivots, k: int | None = None, base: int = 0):
    Dk = _k(D)
    col, colEnd = _k(col), _k(colEnd)
    P = _k(pivots) if len(pivots) else np.zeros(1, np.uint64)
    k = len(pivots) + 1 if k is None else k
    buc = np.zeros(k, np.uint64)
    lib().sqo_initial_bucket_cursors(_p64(Dk), len(col), _p64(col), _p64(colEnd), _p64(P), k,
                                     base, _p64(buc))
    return buc


def naive_skew_transpose(A, col, colEnd, pivots, buc, D=None, vals=None, poff: int = 0,
                         k: int | None = None):
    """Alg 3 on the whole cursor state; returns (D, Dv, col, buc) after the call."""
    Ak, Av = _k(A), _v(vals)
    D = np.zeros(len(Ak), np.uint64) if D is None else _k(D)
    Dv = None if Av is None else np.zeros(len(Ak), np.uint32)
    col, colEnd = _k(col), _k(colEnd)
    P = _k(pivots) if len(pivots) else np.zeros(1, np.uint64)
    buc = _k(buc)
    k = len(buc) if k is None else k
    lib().sqo_naive_skew_transpose(_p64(Ak), _p32(Av), _p64(D), _p32(Dv), len(col), _p64(col),
                                   _p64(colEnd), k, poff, _p64(P), len(pivots), _p64(buc))
    return D, Dv, col, buc


def skew_transpose(A, col, colEnd, pivots, buc, T: int = 4, D=None, vals=None):
    """Alg 2 (recursive, threshold T); returns (D, Dv, col, buc) after the call."""
    Ak, Av = _k(A), _v(vals)
    D = np.zeros(len(Ak), np.uint64) if D is None else _k(D)
    Dv = None if Av is None else np.zeros(len(Ak), np.uint32)
    col, colEnd = _k(col), _k(colEnd)
    P = _k(pivots) if len(pivots) else np.zeros(1, np.uint64)
    buc = _k(buc)
    lib().sqo_skew_transpose(_p64(Ak), _p32(Av), _p64(D), _p32(Dv), len(col), _p64(col),
                             _p64(colEnd), len(buc), 0, _p64(P), len(pivots), _p64(buc), T)
    return D, Dv, col, buc


def _params(cutoff, threshold, cap, sample_from_input):
    return _Params(cutoff, threshold, cap, 1 if sample_from_input else 0)


def square_sort(keys, vals=None, seed: int = 0, cutoff: int = 16, threshold: int = 4,
                cap: int = 32, sample_from_input: bool = False):
    """SquareSort (Alg 1).  Returns (sorted_keys_u64, sorted_vals_or_None, Stats)."""
    A, Av = _k(keys), _v(vals)
    D = np.zeros_like(A)
    Dv = None if Av is None else np.zeros_like(Av)
    st = _Stats()
    prm = _params(cutoff, threshold, cap, sample_from_input)
    rc = lib().sqo_square_sort(_p64(A), _p32(Av), _p64(D), _p32(Dv), len(A), seed & (2**64 - 1),
                               ctypes.byref(prm), ctypes.byref(st))
    if rc != 0:
        raise ValueError("invalid oracle parameters (cutoff >= 4, threshold >= 2, cap >= 1)")
    return D, Dv, Stats(st.nodes, st.rounds, st.degenerate, st.max_depth,
                        st.single_value_buckets)


def level(keys, vals=None, node: int | None = None, seed: int = 0, cutoff: int = 16,
          threshold: int = 4, cap: int = 32, sample_from_input: bool = True):
    """One SquareSort level up to the SkewTranspose.  Returns
    (post_transpose_keys, post_vals, pivots[m-1], bucEnd[m], round, degenerate)."""
    A, Av = _k(keys), _v(vals)
    n = len(A)
    if n <= 4:
        raise ValueError("level() needs n > 4")
    m = ceil_sqrt(n)
    D = np.zeros_like(A)
    Dv = None if Av is None else np.zeros_like(Av)
    P = np.zeros(m - 1, np.uint64)
    be = np.zeros(m, np.uint64)
    deg = ctypes.c_uint32(0)
    node = root_key(seed) if node is None else node
    prm = _params(cutoff, threshold, cap, sample_from_input)
    r = lib().sqo_level(_p64(A), _p32(Av), _p64(D), _p32(Dv), n, node, ctypes.byref(prm),
                        _p64(P), _p64(be), ctypes.byref(deg))
    return A, Av, P, be, int(r), int(deg.value)


def skew_transpose_matrix(src, rows: int, cols: int, pivots, k: int | None = None,
                          n: int | None = None, buc_in=None, T: int = 4, vals=None):
    """The standalone SkewTranspose with the ABI's parameters.
    Returns (dst, dst_vals, buc_out)."""
    S, Sv = _k(src), _v(vals)
    n = len(S) if n is None else n
    k = len(pivots) + 1 if k is None else k
    P = _k(pivots) if len(pivots) else np.zeros(1, np.uint64)
    dst = np.zeros(len(S), np.uint64)
    dv = None if Sv is None else np.zeros(len(S), np.uint32)
    bo = np.zeros(k, np.uint64)
    bi = None if buc_in is None else _k(buc_in)
    lib().sqo_skew_transpose_matrix(_p64(S), _p32(Sv), _p64(dst), _p32(dv), rows, cols, n,
                                    _p64(P), k, _p64(bi), _p64(bo), T)
    return dst, dv, bo


# ----------------------------------------------------------------- signed / IEEE keys
# DESIGN.md reading L25.  The paper sorts integers (P:846,
# P:1048); signed and floating-point keys are sorted by an order-preserving
# bijection onto unsigned keys of the same width -- signed: add 2^(w-1), i.e. flip
# the sign bit; IEEE-754: the totalOrder predicate of IEEE 754-2008 5.10, written
# out as "negative values in reverse bit order below all non-negative values in
# bit order".  These functions are the definition, not a port of the kernel's map.
_UNS = {np.dtype(np.int32): np.uint32, np.dtype(np.int64): np.uint64,
        np.dtype(np.float32): np.uint32, np.dtype(np.float64): np.uint64}


def total_order_key(a):
    """Unsigned key whose unsigned order is the value order of `a` (ints) or the
    IEEE totalOrder of `a` (floats).  Element by element, plain Python ints."""
    a = np.asarray(a)
    u = _UNS[a.dtype]
    w = np.dtype(u).itemsize * 8
    bits = a.view(u)
    out = np.empty(len(a), u)
    for i, b in enumerate(bits.tolist()):
        if a.dtype.kind == "i":
            v = int(a[i])
            out[i] = v + (1 << (w - 1))            # -2^(w-1) .. 2^(w-1)-1  ->  0 .. 2^w-1
        else:
            neg = b >> (w - 1)
            mag = b & ((1 << (w - 1)) - 1)         # |x| as an unsigned bit pattern
            # negatives: larger magnitude first, all below +0; non-negatives above
            out[i] = ((1 << (w - 1)) - 1 - mag) if neg else ((1 << (w - 1)) + mag)
    return out


def from_total_order_key(k, dtype):
    """Inverse of total_order_key."""
    dtype = np.dtype(dtype)
    u = _UNS[dtype]
    w = np.dtype(u).itemsize * 8
    out = np.empty(len(k), u)
    for i, x in enumerate(np.asarray(k, u).tolist()):
        if dtype.kind == "i":
            out[i] = x - (1 << (w - 1)) + (1 << w if x < (1 << (w - 1)) else 0)
        else:
            out[i] = (x - (1 << (w - 1))) if x >= (1 << (w - 1)) else \
                ((1 << (w - 1)) | ((1 << (w - 1)) - 1 - x))
    return out.view(dtype)


def square_sort_mapped(a, seed: int = 0, **kw):
    """SquareSort of signed / float keys: map, Alg 1 on the unsigned keys, unmap."""
    a = np.asarray(a)
    d, _, st = square_sort(total_order_key(a), seed=seed, **kw)
    return from_total_order_key(d.astype(_UNS[a.dtype]), a.dtype), st

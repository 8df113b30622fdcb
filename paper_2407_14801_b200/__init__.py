"""B200-native SquareSort (arXiv 2407.14801): a thin ctypes binding over
libsquaresort.so (include/squaresort.h).  Argument marshalling only -- every
step of the sort runs in the library's CUDA kernels.  PyTorch supplies device
memory (tensor.data_ptr()) and streams; nothing here computes on the data.

There is no CPU fallback: if the library is missing or the device is not a
B200, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# (SQ_LIB_PATH: an experiment build of the same library, for A/B runs)
LIB_PATH = os.environ.get("SQ_LIB_PATH") or os.path.join(_HERE, "libsquaresort.so")
_lib = None

SQ_OK = 0
SQ_FLAG_VALIDATE = 1
STATUS = {0: "SQ_OK", 1: "SQ_ERR_INVALID_ARGUMENT", 2: "SQ_ERR_OUT_OF_MEMORY", 3: "SQ_ERR_CUDA",
          4: "SQ_ERR_PRECONDITION", 5: "SQ_ERR_UNSUPPORTED_DEVICE"}
EXPORTS = ["sq_sort_u32", "sq_sort_u64", "sq_sort_pairs_u32_u32", "sq_sort_u32_host",
           "sq_sort_u64_host", "sq_sort_pairs_u32_u32_host", "sq_sort_u32_host_batch",
           "sq_sort_i32", "sq_sort_i64", "sq_sort_f32", "sq_sort_f64",
           "sq_sort_u64_host_batch", "sq_skew_transpose",
           "sq_status_string", "sq_last_error_message", "sq_get_stats", "sq_set_max_tile",
           "sq_debug_level_u32", "sq_profile", "sq_profile_read", "sq_set_big_bucket_mode",
           "sq_trim_memory", "sq_set_base_case", "sq_debug_level_u64", "sq_sort_pairs_u64_u32",
           "sq_sort_pairs_u64_u32_host", "sq_skew_transpose_u64", "sq_root_key", "sq_draw_positions"]


class SqError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class SkewParams(ctypes.Structure):
    _fields_ = [("pivots", ctypes.c_void_p), ("k", ctypes.c_uint32), ("n", ctypes.c_uint64),
                ("buc_in", ctypes.c_void_p), ("buc_out", ctypes.c_void_p),
                ("naive_threshold", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


class SkewParamsU64(ctypes.Structure):
    _fields_ = [("pivots", ctypes.c_void_p), ("k", ctypes.c_uint32), ("n", ctypes.c_uint64),
                ("buc_in", ctypes.c_void_p), ("buc_out", ctypes.c_void_p),
                ("naive_threshold", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


class Stats(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_uint32), ("kernel_launches", ctypes.c_uint32),
                ("host_syncs", ctypes.c_uint32), ("top_round", ctypes.c_uint32),
                ("top_degenerate", ctypes.c_uint32), ("top_m", ctypes.c_uint32),
                ("oversize_keys", ctypes.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def lib():
    """Load libsquaresort.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2407_14801_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, u64, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint32
        for f in ("sq_sort_u32", "sq_sort_u64", "sq_sort_u32_host", "sq_sort_u64_host", "sq_sort_i32",
                  "sq_sort_i64", "sq_sort_f32", "sq_sort_f64"):
            getattr(L, f).argtypes = [vp, sz, u64, vp]
            getattr(L, f).restype = ctypes.c_int
        for f in ("sq_sort_pairs_u32_u32", "sq_sort_pairs_u32_u32_host", "sq_sort_pairs_u64_u32",
                  "sq_sort_pairs_u64_u32_host"):
            getattr(L, f).argtypes = [vp, vp, sz, u64, vp]
            getattr(L, f).restype = ctypes.c_int
        for f in ("sq_sort_u32_host_batch", "sq_sort_u64_host_batch"):
            getattr(L, f).argtypes = [vp, vp, sz, sz, u64, vp]
            getattr(L, f).restype = ctypes.c_int
        L.sq_skew_transpose.argtypes = [vp, vp, sz, sz, ctypes.POINTER(SkewParams), vp]
        L.sq_skew_transpose.restype = ctypes.c_int
        L.sq_skew_transpose_u64.argtypes = [vp, vp, sz, sz, ctypes.POINTER(SkewParamsU64), vp]
        L.sq_skew_transpose_u64.restype = ctypes.c_int
        L.sq_status_string.argtypes = [ctypes.c_int]
        L.sq_status_string.restype = ctypes.c_char_p
        L.sq_last_error_message.argtypes = []
        L.sq_last_error_message.restype = ctypes.c_char_p
        L.sq_get_stats.argtypes = [ctypes.POINTER(Stats)]
        L.sq_get_stats.restype = None
        L.sq_set_max_tile.argtypes = [u32]
        L.sq_set_max_tile.restype = ctypes.c_int
        L.sq_set_big_bucket_mode.argtypes = [ctypes.c_int]
        L.sq_set_big_bucket_mode.restype = ctypes.c_int
        L.sq_profile.argtypes = [ctypes.c_int]
        L.sq_profile.restype = ctypes.c_int
        L.sq_profile_read.argtypes = [ctypes.c_char_p, sz]
        L.sq_profile_read.restype = ctypes.c_int
        L.sq_debug_level_u32.argtypes = [vp, vp, sz, u64, vp, vp, vp, vp]
        L.sq_debug_level_u32.restype = ctypes.c_int
        L.sq_debug_level_u64.argtypes = [vp, vp, sz, u64, vp, vp, vp, vp]
        L.sq_debug_level_u64.restype = ctypes.c_int
        L.sq_set_base_case.argtypes = [ctypes.c_int]
        L.sq_set_base_case.restype = ctypes.c_int
        L.sq_root_key.argtypes = [u64]
        L.sq_root_key.restype = u64
        L.sq_draw_positions.argtypes = [u64, u32, u32, u64, vp]
        L.sq_draw_positions.restype = ctypes.c_int
        L.sq_trim_memory.argtypes = []
        L.sq_trim_memory.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != SQ_OK:
        raise SqError(rc, lib().sq_last_error_message().decode())


def _stream(stream, device=None):
    if stream is not None:  # a torch.cuda.Stream or a raw cudaStream_t handle
        return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev(t, dtype_name, device=None):
    """data_ptr() of a contiguous CUDA tensor of the given dtype (on `device` if given)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise TypeError("expected a contiguous CUDA tensor")
    if str(t.dtype) != dtype_name:
        raise TypeError(f"expected {dtype_name}, got {t.dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"tensor on {t.device}, expected {device}")
    return ctypes.c_void_p(t.data_ptr())


def _on(t):
    """Run the library call with the tensor's device current (the library works
    on the current device and its stream)."""
    import torch
    return torch.cuda.device(t.device)


def _seed(seed):
    return ctypes.c_uint64(int(seed) & (2**64 - 1))


# ------------------------------------------------------------------ device-buffer calls
def sort_u32(keys, seed: int = 0, stream=None):
    """Sort a contiguous torch.uint32 CUDA tensor in place (sq_sort_u32)."""
    with _on(keys):
        _check(lib().sq_sort_u32(_dev(keys, "torch.uint32"), keys.numel(), _seed(seed), _stream(stream)))
    return keys


def sort_u64(keys, seed: int = 0, stream=None):
    """Sort a contiguous torch.uint64 CUDA tensor in place (sq_sort_u64)."""
    with _on(keys):
        _check(lib().sq_sort_u64(_dev(keys, "torch.uint64"), keys.numel(), _seed(seed), _stream(stream)))
    return keys


def sort_i32(keys, seed: int = 0, stream=None):
    """Sort a contiguous torch.int32 CUDA tensor in place (sq_sort_i32)."""
    with _on(keys):
        _check(lib().sq_sort_i32(_dev(keys, "torch.int32"), keys.numel(), _seed(seed), _stream(stream)))
    return keys


def sort_i64(keys, seed: int = 0, stream=None):
    """Sort a contiguous torch.int64 CUDA tensor in place (sq_sort_i64)."""
    with _on(keys):
        _check(lib().sq_sort_i64(_dev(keys, "torch.int64"), keys.numel(), _seed(seed), _stream(stream)))
    return keys


def sort_f32(keys, seed: int = 0, stream=None):
    """Sort a contiguous torch.float32 CUDA tensor in place by IEEE totalOrder (sq_sort_f32)."""
    with _on(keys):
        _check(lib().sq_sort_f32(_dev(keys, "torch.float32"), keys.numel(), _seed(seed), _stream(stream)))
    return keys


def sort_f64(keys, seed: int = 0, stream=None):
    """Sort a contiguous torch.float64 CUDA tensor in place by IEEE totalOrder (sq_sort_f64)."""
    with _on(keys):
        _check(lib().sq_sort_f64(_dev(keys, "torch.float64"), keys.numel(), _seed(seed), _stream(stream)))
    return keys


def sort_pairs_u32_u32(keys, vals, seed: int = 0, stream=None):
    """Stable sort of (keys, vals) uint32 CUDA tensors by key, in place."""
    if vals.numel() != keys.numel():
        raise ValueError("keys and vals differ in length")
    with _on(keys):
        _check(lib().sq_sort_pairs_u32_u32(_dev(keys, "torch.uint32"), _dev(vals, "torch.uint32", keys.device),
                                           keys.numel(), _seed(seed), _stream(stream)))
    return keys, vals


def sort_pairs_u64_u32(keys, vals, seed: int = 0, stream=None):
    """Stable sort of (torch.uint64 keys, torch.uint32 vals) CUDA tensors by key, in place."""
    if vals.numel() != keys.numel():
        raise ValueError("keys and vals differ in length")
    with _on(keys):
        _check(lib().sq_sort_pairs_u64_u32(_dev(keys, "torch.uint64"), _dev(vals, "torch.uint32", keys.device),
                                           keys.numel(), _seed(seed), _stream(stream)))
    return keys, vals


def skew_transpose(src, dst, rows: int, cols: int, pivots=None, k: int | None = None,
                   n: int = 0, buc_in=None, buc_out=None, naive_threshold: int = 4,
                   flags: int = 0, stream=None):
    """sq_skew_transpose (torch.uint32) or sq_skew_transpose_u64 (torch.uint64) on CUDA
    tensors, all on src's device.  Returns buc_out."""
    import torch
    wide = src.dtype == torch.uint64
    kdt = "torch.uint64" if wide else "torch.uint32"
    k = (pivots.numel() + 1 if pivots is not None else 1) if k is None else k
    dev = src.device
    with _on(src):
        if buc_out is None:
            buc_out = torch.empty(k, dtype=torch.uint32, device=dev)
        kptr = lambda t: _dev(t, kdt, dev) if t is not None and t.numel() else None
        cptr = lambda t: _dev(t, "torch.uint32", dev) if t is not None and t.numel() else None
        P = SkewParamsU64 if wide else SkewParams
        p = P(kptr(pivots), k, n, cptr(buc_in), cptr(buc_out), naive_threshold, flags)
        fn = lib().sq_skew_transpose_u64 if wide else lib().sq_skew_transpose
        _check(fn(kptr(src), kptr(dst), rows, cols, ctypes.byref(p), _stream(stream)))
    return buc_out


def debug_level_u32(src, dst, seed: int, pivots_out, bucend_out, info_out, stream=None):
    d = src.device
    with _on(src):
        _check(lib().sq_debug_level_u32(_dev(src, "torch.uint32"), _dev(dst, "torch.uint32", d),
                                        src.numel(), _seed(seed), _dev(pivots_out, "torch.uint32", d),
                                        _dev(bucend_out, "torch.uint32", d), _dev(info_out, "torch.uint32", d),
                                        _stream(stream)))


def debug_level_u64(src, dst, seed: int, pivots_out, bucend_out, info_out, stream=None):
    d = src.device
    with _on(src):
        _check(lib().sq_debug_level_u64(_dev(src, "torch.uint64"), _dev(dst, "torch.uint64", d),
                                        src.numel(), _seed(seed), _dev(pivots_out, "torch.uint64", d),
                                        _dev(bucend_out, "torch.uint32", d), _dev(info_out, "torch.uint32", d),
                                        _stream(stream)))


# ------------------------------------------------------------------ host-buffer calls
def _host_ptr(a, dtype):
    import numpy as np
    if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous):
        raise TypeError(f"expected a contiguous numpy {dtype} array")
    return ctypes.c_void_p(a.ctypes.data)


def sort_u32_host(keys, seed: int = 0, stream=None):
    import numpy as np
    _check(lib().sq_sort_u32_host(_host_ptr(keys, np.uint32), keys.size, _seed(seed), _stream(stream)))
    return keys


def sort_u64_host(keys, seed: int = 0, stream=None):
    import numpy as np
    _check(lib().sq_sort_u64_host(_host_ptr(keys, np.uint64), keys.size, _seed(seed), _stream(stream)))
    return keys


def sort_pairs_u32_u32_host(keys, vals, seed: int = 0, stream=None):
    import numpy as np
    _check(lib().sq_sort_pairs_u32_u32_host(_host_ptr(keys, np.uint32), _host_ptr(vals, np.uint32),
                                            keys.size, _seed(seed), _stream(stream)))
    return keys, vals


def sort_pairs_u64_u32_host(keys, vals, seed: int = 0, stream=None):
    import numpy as np
    _check(lib().sq_sort_pairs_u64_u32_host(_host_ptr(keys, np.uint64), _host_ptr(vals, np.uint32),
                                            keys.size, _seed(seed), _stream(stream)))
    return keys, vals


def _host_batch(fn, ins, outs, dtype, seed, stream):
    if len(ins) != len(outs):
        raise ValueError("ins and outs differ in length")
    n = ins[0].size if ins else 0
    for a in list(ins) + list(outs):
        _host_ptr(a, dtype)
        if a.size != n:
            raise ValueError("all batch items must have the same length")
    arr = ctypes.c_void_p * max(1, len(ins))
    pi = arr(*[a.ctypes.data for a in ins])
    po = arr(*[a.ctypes.data for a in outs])
    _check(fn(pi, po, n, len(ins), _seed(seed), _stream(stream)))
    return outs


def sort_u32_host_batch(ins, outs, seed: int = 0, stream=None):
    """Pipelined batch: outs[i] <- sorted(ins[i]) (numpy uint32 arrays, ideally pinned)."""
    import numpy as np
    return _host_batch(lib().sq_sort_u32_host_batch, ins, outs, np.uint32, seed, stream)


def sort_u64_host_batch(ins, outs, seed: int = 0, stream=None):
    import numpy as np
    return _host_batch(lib().sq_sort_u64_host_batch, ins, outs, np.uint64, seed, stream)


# ------------------------------------------------------------------ sampler RNG (host)
def root_key(seed: int) -> int:
    return int(lib().sq_root_key(_seed(seed)))


def draw_positions(node: int, rounds: int, count: int, n: int):
    """numpy uint64 [rounds, count]: the sample positions of a level of n keys (sq_draw_positions)."""
    import numpy as np
    out = np.zeros((rounds, count), np.uint64)
    _check(lib().sq_draw_positions(ctypes.c_uint64(node), rounds, count, n, ctypes.c_void_p(out.ctypes.data)))
    return out


# ------------------------------------------------------------------ introspection
def get_stats() -> dict:
    s = Stats()
    lib().sq_get_stats(ctypes.byref(s))
    return s.as_dict()


def set_max_tile(t: int):
    _check(lib().sq_set_max_tile(t))


BIG_LEVEL, BIG_MERGE, BIG_CLUSTER, BIG_BINCLUSTER, BIG_SPLIT = 0, 1, 2, 3, 4


def set_big_bucket_mode(mode: int):
    """0: recurse into a SquareSort level, 1: multi-CTA merge sort (default), 2: clusters
    merging through DSMEM, 3: clusters of counting-sort tiles (u32 keys; others: 1)."""
    _check(lib().sq_set_big_bucket_mode(mode))


BASE_MERGE, BASE_BIN = 0, 1


def set_base_case(which: int):
    """On-chip base case of keys-only u32 sorts: 1 counting sort + fix-up (default), 0 merge sort."""
    _check(lib().sq_set_base_case(which))


def trim_memory():
    """Return the scratch the library's pool keeps on the current device (sq_trim_memory)."""
    _check(lib().sq_trim_memory())


def profile(enable: bool = True):
    """Enable/disable per-kernel CUDA-event timing inside the library."""
    _check(lib().sq_profile(1 if enable else 0))


def profile_read() -> dict:
    """{role: (launches, total_ms)} accumulated since the last read."""
    import json
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().sq_profile_read(buf, len(buf)))
    return {k: (int(v[0]), float(v[1])) for k, v in json.loads(buf.value.decode()).items()}

"""The C-ABI library loads and exports every symbol include/squaresort.h declares
(no compute calls -- this runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "squaresort.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2407_14801_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("sq_sort_u32", "sq_sort_u64", "sq_sort_pairs_u32_u32", "sq_skew_transpose"):
        assert f in names


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared_functions()) <= exported


def test_python_binding_lists_exports(libpath):
    import paper_2407_14801_b200 as sq
    assert set(sq.EXPORTS) == set(declared_functions())


def test_status_strings_without_gpu(libpath):
    import paper_2407_14801_b200 as sq
    L = sq.lib()
    for code, name in sq.STATUS.items():
        assert L.sq_status_string(code).decode() == name


def test_argument_errors_without_gpu(libpath):
    # argument validation happens before any CUDA call
    import paper_2407_14801_b200 as sq
    L = sq.lib()
    assert L.sq_sort_u32(None, 10, 0, None) == 1
    assert L.sq_sort_u32(None, 0, 0, None) == 0  # n = 0 is a no-op
    assert L.sq_sort_u32(None, 1, 0, None) == 0
    assert L.sq_sort_pairs_u32_u32(ctypes.c_void_p(4096), None, 10, 0, None) == 1
    assert L.sq_sort_pairs_u32_u32(ctypes.c_void_p(4096), ctypes.c_void_p(4100), 10, 0, None) == 1
    assert L.sq_sort_u32(ctypes.c_void_p(4096), (1 << 30) + 1, 0, None) == 1
    p = sq.SkewParams(None, 0, 0, None, None, 4, 0)
    assert L.sq_skew_transpose(None, None, 4, 4, ctypes.byref(p), None) == 1  # k = 0
    p = sq.SkewParams(None, 1, 0, None, ctypes.c_void_p(64), 1, 0)
    assert L.sq_skew_transpose(None, None, 4, 4, ctypes.byref(p), None) == 1  # threshold 1
    p = sq.SkewParams(None, 1, 17, None, ctypes.c_void_p(64), 4, 0)
    assert L.sq_skew_transpose(ctypes.c_void_p(4096), ctypes.c_void_p(1 << 20), 4, 4,
                               ctypes.byref(p), None) == 1  # n > rows*cols
    p = sq.SkewParams(None, 3, 0, None, ctypes.c_void_p(64), 4, 0)
    assert L.sq_skew_transpose(ctypes.c_void_p(4096), ctypes.c_void_p(1 << 20), 4, 4,
                               ctypes.byref(p), None) == 1  # NULL pivots with k > 1
    p = sq.SkewParams(None, 1, 0, None, ctypes.c_void_p(64), 4, 0)
    assert L.sq_skew_transpose(ctypes.c_void_p(4096), ctypes.c_void_p(4100), 4, 4,
                               ctypes.byref(p), None) == 1  # overlap
    arr = ctypes.c_void_p * 2
    a, b = arr(4096, 1 << 20), arr(1 << 24, (1 << 24) + 64)
    assert L.sq_sort_u32_host_batch(a, b, 10, 0, 0, None) == 0  # count = 0 is a no-op
    assert L.sq_sort_u32_host_batch(None, b, 10, 2, 0, None) == 1
    assert L.sq_sort_u32_host_batch(a, arr(1 << 24, 0), 10, 2, 0, None) == 1  # NULL item
    assert L.sq_sort_u64_host_batch(a, arr((1 << 20) + 8, 1 << 24), 10, 2, 0, None) == 1  # out[0] overlaps in[1]
    assert L.sq_sort_u32_host(None, 10, 0, None) == 1
    assert L.sq_set_max_tile(100) == 1 and L.sq_set_max_tile(0) == 0
    assert L.sq_last_error_message() is not None


def test_no_oracle_on_the_product_path():
    # The product package never imports, includes or loads the oracle.
    pkg = os.path.join(ROOT, "paper_2407_14801_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "squaresort_oracle",
                            "sqo_", "numpy.sort", "np.sort"):
                    assert bad not in txt, (f, bad)

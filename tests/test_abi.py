"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol that
include/sketch.h declares, and rejects bad arguments before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sketch.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sketch_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2310_15419_b200 import sketch
    return sketch.load_library()


def test_header_declares_the_north_star_entry_points():
    names = _declared_functions()
    for must in ("sketch_plan", "sketch_apply", "sketch_apply_csc", "sketch_fill_s",
                 "sketch_plan_stats", "sketch_plan_destroy", "sketch_error_string"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2310_15419_b200 import sketch
    names = _declared_functions()
    assert set(names) == set(sketch.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name


def test_error_strings_and_version(lib):
    assert lib.sketch_error_string(0) == b"ok"
    assert lib.sketch_error_string(-2) == b"CSC validation failed"
    assert lib.sketch_error_string(-99) == b"unknown status"
    assert lib.sketch_version().startswith(b"libsketch")


def test_argument_validation_happens_before_any_device_work(lib):
    from paper_2310_15419_b200 import sketch as sk
    # bad enums, bad ranges, NULL outputs: all rejected on the host with SK_EINVAL
    assert lib.sketch_fill_s(1, 7, 0, 0, 4, 0, 4, ctypes.c_void_p(1), 4, None) == sk.SK_EINVAL
    assert lib.sketch_fill_s(1, 0, 5, 0, 4, 0, 4, ctypes.c_void_p(1), 4, None) == sk.SK_EINVAL
    assert lib.sketch_fill_s(1, 0, 0, 4, 0, 0, 4, ctypes.c_void_p(1), 4, None) == sk.SK_EINVAL   # i1 < i0
    assert lib.sketch_fill_s(1, 0, 0, 0, 8, 0, 4, ctypes.c_void_p(1), 4, None) == sk.SK_EINVAL   # ld < rows
    assert lib.sketch_fill_s(1, 0, 0, 0, 8, 0, 4, None, 8, None) == sk.SK_EINVAL                 # NULL out
    assert lib.sketch_fill_s(1, 0, 0, 0, 0, 0, 4, None, 0, None) == sk.SK_OK                     # empty: no-op
    assert lib.sketch_plan(None, 0, 10, 10, 1, 0, None, None, 0, None) == sk.SK_EINVAL
    h = ctypes.c_void_p()
    assert lib.sketch_plan(ctypes.byref(h), 0, 0, 10, 1, 0, ctypes.c_void_p(1), None, 0, None) == sk.SK_EINVAL  # d < 1
    assert lib.sketch_plan(ctypes.byref(h), 3, 10, 10, 1, 0, ctypes.c_void_p(1), None, 0, None) == sk.SK_EINVAL  # dtype
    assert lib.sketch_plan(ctypes.byref(h), 0, 2**31, 10, 1, 0, ctypes.c_void_p(1), None, 0, None) == sk.SK_EINVAL
    assert lib.sketch_plan(ctypes.byref(h), 0, 10, 10, 1, -1, ctypes.c_void_p(1), None, 0, None) == sk.SK_EINVAL
    assert h.value is None
    assert lib.sketch_apply(None, 1, 0, None, None, None) == sk.SK_EINVAL
    assert lib.sketch_plan_destroy(None) == sk.SK_OK
    assert lib.sketch_plan_stats(None, None) == sk.SK_EINVAL


def test_kernel_selectors_validate_on_host(lib):
    # the process-wide selectors take only their documented values (no device work)
    from paper_2310_15419_b200 import sketch as sk
    for bad in (-2, 2, 7):
        assert lib.sketch_set_f4_persistent(bad) == sk.SK_EINVAL
    for bad in (1, 2, 4, -1):
        assert lib.sketch_set_rad_f64_path(bad) == sk.SK_EINVAL
    for bad in (3, -1):
        assert lib.sketch_set_pair_path(bad) == sk.SK_EINVAL
    for good in (-1, 0, 1):
        assert lib.sketch_set_f4_persistent(good) == sk.SK_OK
    assert lib.sketch_set_f4_persistent(-1) == sk.SK_OK       # back to auto
    with pytest.raises(KeyError):
        sk.set_f4_persistent("sometimes")


def test_host_entry_point_validates_colptr_on_host(lib):
    import numpy as np
    from paper_2310_15419_b200 import sketch as sk
    bad = np.array([0, 3, 2], dtype=np.int64)        # decreasing colptr
    rows = np.zeros(2, dtype=np.int32)
    vals = np.zeros(2)
    out = np.zeros((2, 4))
    rc = lib.sketch_apply_host(1, 0, 0, 4, 10, 2, 0, bad.ctypes.data, rows.ctypes.data,
                               vals.ctypes.data, out.ctypes.data, 0, None)
    assert rc == sk.SK_ECSC
    nz = np.array([1, 2, 2], dtype=np.int64)         # colptr[0] != 0
    rc = lib.sketch_apply_host(1, 0, 0, 4, 10, 2, 0, nz.ctypes.data, rows.ctypes.data,
                               vals.ctypes.data, out.ctypes.data, 0, None)
    assert rc == sk.SK_ECSC
    rc = lib.sketch_apply_host(1, 9, 0, 4, 10, 2, 0, nz.ctypes.data, rows.ctypes.data,
                               vals.ctypes.data, out.ctypes.data, 0, None)
    assert rc == sk.SK_EINVAL


def test_product_path_has_no_oracle_or_cpu_fallback():
    # the product package must not import the oracle, and must fail loudly without the .so
    pkg = os.path.join(ROOT, "paper_2310_15419_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
    from paper_2310_15419_b200 import sketch
    with pytest.raises(ImportError):
        sketch._open_library(os.path.join(ROOT, "does_not_exist", "libsketch.so"))

"""CPU oracle for the sketch Â = S·A (arXiv 2310.15419) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the product
path (``paper_2310_15419_b200``); see ``sketch_oracle.c`` for the definitions it follows
and the PAPER.md passages each one cites.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py`` against
something other than itself (an independent Philox implementation, closed forms, moments,
brute-force dense products, exact special cases).  See DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sketch_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC"]

RADEMACHER, UNIFORM, GAUSSIAN = 0, 1, 2
F64, F32 = 0, 1
DISTS = {"rademacher": RADEMACHER, "uniform": UNIFORM, "gaussian": GAUSSIAN, "uniform24": 3}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            u32p = ctypes.POINTER(ctypes.c_uint32)
            dp = ctypes.POINTER(ctypes.c_double)
            lib.or_philox4x32_10.argtypes = [u32p, u32p, u32p]
            lib.or_philox4x32_10.restype = None
            lib.or_s_entry_f64.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
            lib.or_s_entry_f64.restype = ctypes.c_double
            lib.or_s_entry.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int64, ctypes.c_int64]
            lib.or_s_entry.restype = ctypes.c_double
            lib.or_get_samples.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int64, dp]
            lib.or_get_samples.restype = None
            lib.or_fill_s.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, dp]
            lib.or_fill_s.restype = ctypes.c_int
            lib.or_sketch.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.or_sketch.restype = ctypes.c_int
            lib.or_max_threads.argtypes = []
            lib.or_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _dist(dist) -> int:
    return DISTS[dist] if isinstance(dist, str) else int(dist)


def _dtype(dtype) -> int:
    if isinstance(dtype, str):
        return {"f64": F64, "float64": F64, "f32": F32, "float32": F32}[dtype]
    if dtype in (np.float64,):
        return F64
    if dtype in (np.float32,):
        return F32
    return int(dtype)


def philox4x32_10(ctr, key) -> tuple:
    """Philox4x32-10 of one counter (4 x u32) under one key (2 x u32)."""
    lib = _load()
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib.or_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def s_entry(seed: int, dist, i: int, j: int, dtype=F64) -> float:
    """S[i, j] by the entry-wise definition (R1-R5)."""
    return _load().or_s_entry(int(seed), _dist(dist), _dtype(dtype), int(i), int(j))


def get_samples(seed: int, dist, j: int, d: int, dtype=F64) -> np.ndarray:
    """Algorithm 3: S[0:d, j] generated block by block."""
    v = np.empty(int(d), dtype=np.float64)
    _load().or_get_samples(int(seed), _dist(dist), _dtype(dtype), int(j), int(d),
                           v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return v


def fill_s(seed: int, dist, i0: int, i1: int, j0: int, j1: int, dtype=F64) -> np.ndarray:
    """S[i0:i1, j0:j1] as a (i1-i0) x (j1-j0) fp64 array (entries of fp32 S widened exactly)."""
    out = np.empty((int(j1) - int(j0), int(i1) - int(i0)), dtype=np.float64)  # column-major
    rc = _load().or_fill_s(int(seed), _dist(dist), _dtype(dtype), int(i0), int(i1), int(j0),
                           int(j1), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError(f"or_fill_s rc={rc}")
    return out.T


def sketch(seed: int, dist, d: int, m: int, n: int, colptr, rowidx, vals, *, dtype=None,
           row_offset: int = 0, threads: int = 1, want_bound: bool = True):
    """Algorithm 3 (kji) sketch.  Returns (Â, B) as d x n fp64 arrays, B = |S|·|A|.

    ``vals`` may be fp64 or fp32; fp32 values are widened exactly and S is rounded to
    fp32 (R5) unless ``dtype`` says otherwise.
    """
    vals = np.asarray(vals)
    if dtype is None:
        dtype = F32 if vals.dtype == np.float32 else F64
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    v64 = np.ascontiguousarray(vals, dtype=np.float64)
    out = np.empty((int(n), int(d)), dtype=np.float64)
    bnd = np.empty((int(n), int(d)), dtype=np.float64) if want_bound else None
    rc = _load().or_sketch(int(seed), _dist(dist), _dtype(dtype), int(d), int(m), int(n),
                           int(row_offset), colptr.ctypes.data, rowidx.ctypes.data,
                           v64.ctypes.data, out.ctypes.data,
                           bnd.ctypes.data if bnd is not None else None, int(threads))
    if rc != 0:
        raise ValueError(f"or_sketch rc={rc}")
    return out.T, (bnd.T if bnd is not None else None)


def max_threads() -> int:
    return int(_load().or_max_threads())

"""Thin ctypes binding to libsketch.so (include/sketch.h) -- argument marshalling only.

Every step of the sketch runs in the library's sm_100a kernels; this module only turns
torch tensors / numpy arrays into pointers, sizes and streams.  There is no CPU fallback:
if ``libsketch.so`` is missing or no CUDA device is present the calls raise.

Names follow the C ABI: ``sketch_plan``, ``sketch_apply``, ``sketch_apply_csc``,
``sketch_apply_host``, ``sketch_fill_s``, ``sketch_plan_stats``, ``sketch_plan_destroy``.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKETCH_LIB") or os.path.join(_HERE, "libsketch.so")   # override: experiments only

RADEMACHER, UNIFORM, GAUSSIAN, UNIFORM24 = 0, 1, 2, 3
F64, F32 = 0, 1
DIST = {"rademacher": RADEMACHER, "uniform": UNIFORM, "gaussian": GAUSSIAN, "uniform24": UNIFORM24}
DTYPE = {"f64": F64, "f32": F32}

SK_OK, SK_EINVAL, SK_ECSC, SK_ENOMEM, SK_ECUDA, SK_EUNSUPPORTED = 0, -1, -2, -3, -4, -5

EXPORTS = ["sketch_plan", "sketch_plan_host", "sketch_apply", "sketch_apply_csc",
           "sketch_apply_host", "sketch_fill_s", "sketch_plan_stats", "sketch_plan_destroy",
           "sketch_error_string", "sketch_last_error_detail", "sketch_version",
           "sketch_set_rad_f64_path", "sketch_apply_kernel_name", "sketch_set_pair_path",
           "sketch_plan_host_jki", "sketch_set_f4_persistent"]
RAD_F64_PATHS = {"fp4": 0, "simt": 3}
PAIR_PATHS = {"auto": 0, "kji": 1, "jki": 2}
_STRING_RESULTS = ("sketch_error_string", "sketch_last_error_detail", "sketch_version",
                   "sketch_apply_kernel_name")


class SketchError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str = ""):
        self.code = code
        super().__init__(f"{where}: {code} ({detail})")


class sk_stats_t(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in
                ("d", "m", "n", "nnz", "row_offset", "max_col_nnz", "n_items_rad", "n_items_pair",
                 "philox_blocks_rad", "philox_blocks_pair", "plan_bytes", "n_items_jki", "jki_nonzero_rows", "n_items_f4_split",
                 "n_items_f4", "n_cols_f4", "jki_block_cols", "f4_persistent")]


_lock = threading.Lock()
_lib = None


def _open_library(path: str):
    if not os.path.exists(path):
        raise ImportError(f"libsketch.so not built at {path}; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    return ctypes.CDLL(path)


def load_library(path: str = LIB_PATH):
    """Load libsketch.so and declare its prototypes (no GPU needed to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = _open_library(path)
        vp, i64, u64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        lib.sketch_plan.argtypes = [ctypes.POINTER(vp), i32, i64, i64, i64, i64, vp, vp, i64, vp]
        lib.sketch_plan_host.argtypes = [ctypes.POINTER(vp), i32, i64, i64, i64, i64, vp, vp, i64,
                                         i32, vp]
        lib.sketch_apply.argtypes = [vp, u64, i32, vp, vp, vp]
        lib.sketch_apply_csc.argtypes = [u64, i32, i32, i64, i64, i64, i64, vp, vp, i64, vp, vp, vp]
        lib.sketch_apply_host.argtypes = [u64, i32, i32, i64, i64, i64, i64, vp, vp, vp, vp, i32, vp]
        lib.sketch_fill_s.argtypes = [u64, i32, i32, i64, i64, i64, i64, vp, i64, vp]
        lib.sketch_plan_stats.argtypes = [vp, ctypes.POINTER(sk_stats_t)]
        lib.sketch_plan_destroy.argtypes = [vp]
        lib.sketch_error_string.argtypes = [i32]
        lib.sketch_error_string.restype = ctypes.c_char_p
        lib.sketch_last_error_detail.argtypes = []
        lib.sketch_last_error_detail.restype = ctypes.c_char_p
        lib.sketch_version.argtypes = []
        lib.sketch_version.restype = ctypes.c_char_p
        lib.sketch_set_rad_f64_path.argtypes = [i32]
        lib.sketch_set_f4_persistent.argtypes = [i32]
        lib.sketch_set_pair_path.argtypes = [i32]
        lib.sketch_plan_host_jki.argtypes = [ctypes.POINTER(vp), i32, i64, i64, i64, i64, vp, vp, i64, i32, vp]
        lib.sketch_apply_kernel_name.argtypes = [vp, i32]
        lib.sketch_apply_kernel_name.restype = ctypes.c_char_p
        for name in EXPORTS:
            if name not in _STRING_RESULTS:
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def _check(rc: int, where: str):
    if rc != SK_OK:
        lib = load_library()
        detail = lib.sketch_error_string(rc).decode()
        extra = lib.sketch_last_error_detail().decode()
        raise SketchError(rc, where, detail + (f"; {extra}" if extra and rc == SK_ECUDA else ""))


def _dist(dist) -> int:
    return DIST[dist] if isinstance(dist, str) else int(dist)


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dtype_of(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"values must be float64 or float32, got {t.dtype}")


def _require_cuda(*tensors):
    for t in tensors:
        if not t.is_cuda:
            raise ValueError("libsketch entry points take device tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")


class Plan:
    """Owning wrapper of an ``sk_plan_t`` built by ``sketch_plan``."""

    def __init__(self, colptr, rowidx, d: int, m: int, dtype="f64", row_offset: int = 0,
                 stream=None, jki: bool = False):
        """``jki=True`` always builds the Algorithm 4 structure (sketch_plan_host_jki); otherwise
        the plan builds it only when a sample shows enough row reuse."""
        import torch
        _require_cuda(colptr, rowidx)
        if colptr.dtype != torch.int64 or rowidx.dtype != torch.int32:
            raise TypeError("colptr must be int64 and rowidx int32")
        lib = load_library()
        self.d, self.m, self.n = int(d), int(m), int(colptr.numel() - 1)
        self.nnz = int(rowidx.numel())
        self.dtype = DTYPE[dtype] if isinstance(dtype, str) else int(dtype)
        self.row_offset = int(row_offset)
        self._keep = (colptr, rowidx)     # the plan references these device buffers
        h = ctypes.c_void_p()
        if jki:
            hc = colptr.cpu().contiguous()
            _check(lib.sketch_plan_host_jki(ctypes.byref(h), self.dtype, self.d, self.m, self.n, self.row_offset,
                                            ctypes.c_void_p(hc.data_ptr()), ctypes.c_void_p(rowidx.data_ptr()),
                                            self.nnz, 1, _stream_ptr(stream)), "sketch_plan_host_jki")
        else:
            _check(lib.sketch_plan(ctypes.byref(h), self.dtype, self.d, self.m, self.n, self.row_offset,
                                   ctypes.c_void_p(colptr.data_ptr()), ctypes.c_void_p(rowidx.data_ptr()),
                                   self.nnz, _stream_ptr(stream)), "sketch_plan")
        self._h = h

    def stats(self) -> dict:
        s = sk_stats_t()
        _check(load_library().sketch_plan_stats(self._h, ctypes.byref(s)), "sketch_plan_stats")
        return {name: int(getattr(s, name)) for name, _ in sk_stats_t._fields_}

    def apply(self, vals, seed: int, dist, out=None, stream=None):
        """Â = S·A as an (n, d) tensor whose transpose ``.T`` is the d x n sketch
        (column-major storage, ld = d).  ``out`` (same shape) is overwritten if given."""
        import torch
        _require_cuda(vals)
        if _dtype_of(vals) != self.dtype or vals.numel() != self.nnz:
            raise ValueError("vals dtype / length does not match the plan")
        if out is None:
            out = torch.empty((self.n, self.d), dtype=vals.dtype, device=vals.device)
        _require_cuda(out)
        if out.shape != (self.n, self.d) or out.dtype != vals.dtype:
            raise ValueError("out must be an (n, d) tensor of the values' dtype")
        _check(load_library().sketch_apply(self._h, int(seed) & (2**64 - 1), _dist(dist),
                                           ctypes.c_void_p(vals.data_ptr()),
                                           ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
               "sketch_apply")
        return out

    def kernel_name(self, dist) -> str:
        """Name of the kernel ``apply`` launches for ``dist``."""
        return load_library().sketch_apply_kernel_name(self._h, _dist(dist)).decode()

    def close(self):
        if getattr(self, "_h", None):
            _check(load_library().sketch_plan_destroy(self._h), "sketch_plan_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sketch_plan(colptr, rowidx, d, m, dtype="f64", row_offset=0, stream=None) -> Plan:
    return Plan(colptr, rowidx, d, m, dtype, row_offset, stream)


def sketch_apply(plan: Plan, vals, seed, dist, out=None, stream=None):
    return plan.apply(vals, seed, dist, out, stream)


def sketch_apply_csc(seed, dist, d, m, colptr, rowidx, vals, out=None, row_offset=0, stream=None):
    """One-shot plan + apply + destroy (the north-star signature).  Returns (n, d) storage."""
    import torch
    _require_cuda(colptr, rowidx, vals)
    n = colptr.numel() - 1
    if out is None:
        out = torch.empty((n, int(d)), dtype=vals.dtype, device=vals.device)
    _check(load_library().sketch_apply_csc(int(seed) & (2**64 - 1), _dist(dist), _dtype_of(vals),
                                           int(d), int(m), int(n), int(row_offset),
                                           ctypes.c_void_p(colptr.data_ptr()),
                                           ctypes.c_void_p(rowidx.data_ptr()), int(rowidx.numel()),
                                           ctypes.c_void_p(vals.data_ptr()),
                                           ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
           "sketch_apply_csc")
    return out


def sketch_apply_host(seed, dist, d, m, colptr, rowidx, vals, out=None, row_offset=0,
                      pipeline_chunks=0, stream=None):
    """End-to-end form with HOST buffers (numpy arrays or CPU tensors, ideally pinned).
    Returns the (n, d) array holding Â column-major: a host array, or ``out`` itself when it is a
    CUDA tensor (the result then stays on the device, e.g. for a cross-GPU reduction)."""
    def _np(x):
        return x.numpy() if hasattr(x, "numpy") and not isinstance(x, np.ndarray) else np.asarray(x)
    cp, ri, va = _np(colptr), _np(rowidx), _np(vals)
    if cp.dtype != np.int64 or ri.dtype != np.int32 or va.dtype not in (np.float64, np.float32):
        raise TypeError("colptr int64, rowidx int32, vals float64/float32")
    for a in (cp, ri, va):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("host arrays must be contiguous")
    n = cp.shape[0] - 1
    if out is None:
        out = np.empty((n, int(d)), dtype=va.dtype)
    if getattr(out, "is_cuda", False):
        if tuple(out.shape) != (n, int(d)) or not out.is_contiguous() or out.element_size() != va.itemsize:
            raise ValueError("out must be a contiguous (n, d) tensor of the values' dtype")
        optr = out.data_ptr()
    else:
        o = _np(out)
        if o.shape != (n, int(d)) or o.dtype != va.dtype or not o.flags["C_CONTIGUOUS"]:
            raise ValueError("out must be a contiguous (n, d) array of the values' dtype")
        optr = o.ctypes.data
    _check(load_library().sketch_apply_host(int(seed) & (2**64 - 1), _dist(dist),
                                            F64 if va.dtype == np.float64 else F32, int(d), int(m),
                                            int(n), int(row_offset), cp.ctypes.data, ri.ctypes.data,
                                            va.ctypes.data, optr, int(pipeline_chunks),
                                            _stream_ptr(stream)), "sketch_apply_host")
    return out


def sketch_fill_s(seed, dist, i0, i1, j0, j1, dtype="f64", device="cuda", stream=None):
    """S[i0:i1, j0:j1] (global indices) as a (j1-j0, i1-i0) tensor = column-major S block."""
    import torch
    dt = DTYPE[dtype] if isinstance(dtype, str) else int(dtype)
    out = torch.empty((int(j1) - int(j0), int(i1) - int(i0)),
                      dtype=torch.float64 if dt == F64 else torch.float32, device=device)
    _check(load_library().sketch_fill_s(int(seed) & (2**64 - 1), _dist(dist), dt, int(i0), int(i1),
                                        int(j0), int(j1), ctypes.c_void_p(out.data_ptr()),
                                        int(i1) - int(i0), _stream_ptr(stream)), "sketch_fill_s")
    return out


def set_rad_f64_path(path) -> None:
    """Select the kernel for ±1 sketches of fp64 values in plans built from now on: "fp4" (tensor
    cores for columns of 896 (1280 for a single wave of items) .. 131071 nonzeros, SIMT for the rest;
    default) or "simt" (process-wide)."""
    p = RAD_F64_PATHS[path] if isinstance(path, str) else int(path)
    _check(load_library().sketch_set_rad_f64_path(p), "sketch_set_rad_f64_path")


def set_f4_persistent(mode) -> None:
    """Tensor-core columns of plans built from now on: "auto" (persistent kernel when there are more
    items than SMs; default), "off" (one CTA per item) or "on" (persistent)."""
    m = {"auto": -1, "off": 0, "on": 1}[mode] if isinstance(mode, str) else int(mode)
    _check(load_library().sketch_set_f4_persistent(m), "sketch_set_f4_persistent")


def set_pair_path(path) -> None:
    """Uniform / Gaussian kernel: "auto" (Algorithm 4 when the plan built it), "kji", "jki"."""
    p = PAIR_PATHS[path] if isinstance(path, str) else int(path)
    _check(load_library().sketch_set_pair_path(p), "sketch_set_pair_path")


def version() -> str:
    return load_library().sketch_version().decode()

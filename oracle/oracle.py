"""Parity oracle - TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product path (``paper_1107_4958_b200``) never
does, and fails loudly when its CUDA library is missing instead of falling back
to anything here.

Two restatements of the reference running-sum filter
(``/root/reference/pkg/src/sliceblur/filtering.py``):

* the C oracle (``sliceblur_oracle.c``, bound with ctypes) - op-for-op float64,
  bit-identical to the reference (pinned against ``tests/golden``);
* a numpy port (``np_filter_rows`` / ``np_separable_filter_2d``) that performs
  the reference's own numpy operations (filtering.py:48-64, 76-104), so it runs
  at the reference's speed; ``bench.py --impl reference`` times it with a
  thread pool over row blocks exactly like the reference's ``parallel=True``
  (filtering.py:91-101) but on every host core.

Parity pinned: every function here is checked bit-for-bit against the
reference's outputs in ``tests/golden/filter_cases.npz`` (tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libsliceblur_oracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile the C oracle with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_filter_rows.argtypes = [_f64p, _f64p, ctypes.c_int64, ctypes.c_int64, _i64p, _f64p, ctypes.c_int,
                                           ctypes.c_int]
        lib.oracle_filter_rows.restype = ctypes.c_int
        lib.oracle_separable_2d.argtypes = [_f64p, _f64p, _f64p, ctypes.c_int64, ctypes.c_int64, _i64p, _f64p,
                                            ctypes.c_int, ctypes.c_int]
        lib.oracle_separable_2d.restype = ctypes.c_int
        lib.oracle_prefix_sum.argtypes = [_f64p, _f64p, ctypes.c_int64]
        lib.oracle_prefix_sum.restype = None
        lib.oracle_filter_at.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, _i64p, _f64p, ctypes.c_int, _i64p,
                                         _i64p, ctypes.c_int64, _f64p, _f64p, _f64p, _f64p]
        lib.oracle_filter_at.restype = ctypes.c_int
        lib.oracle_filter_columns.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, _i64p, _f64p, ctypes.c_int, _i64p, ctypes.c_int64,
                                              _f64p, _f64p, ctypes.c_int]
        lib.oracle_filter_columns.restype = ctypes.c_int
        lib.oracle_filter_band.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, _i64p, _f64p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                           _f64p, _f64p, ctypes.c_int]
        lib.oracle_filter_band.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p64(a):
    return a.ctypes.data_as(_f64p)


def _pi64(a):
    return a.ctypes.data_as(_i64p)


def _kernel_arrays(radii, weights):
    r = np.ascontiguousarray(radii, dtype=np.int64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if r.ndim != 1 or r.shape != w.shape or r.size == 0:
        raise ValueError("radii/weights must be equal-length 1D arrays")
    return r, w


def filter_rows(arr, radii, weights, threads: int = 1) -> np.ndarray:
    """C restatement of ``_filter_rows`` (filtering.py:48-64) on a 2D array."""
    a = np.ascontiguousarray(arr, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("need a 2D array")
    r, w = _kernel_arrays(radii, weights)
    out = np.empty_like(a)
    if _load().oracle_filter_rows(_p64(a), _p64(out), a.shape[0], a.shape[1], _pi64(r), _p64(w), r.size, threads):
        raise MemoryError("oracle_filter_rows failed")
    return out


def separable_filter_2d(image, radii, weights, threads: int = 1) -> np.ndarray:
    """C restatement of ``separable_filter_2d`` (filtering.py:76-104), no validation."""
    a = np.ascontiguousarray(image, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("need a 2D image")
    r, w = _kernel_arrays(radii, weights)
    out = np.empty_like(a)
    tmp = np.empty_like(a)
    if _load().oracle_separable_2d(_p64(a), _p64(out), _p64(tmp), a.shape[0], a.shape[1], _pi64(r), _p64(w), r.size,
                                   threads):
        raise MemoryError("oracle_separable_2d failed")
    return out


def prefix_sum(values) -> np.ndarray:
    """C restatement of ``prefix_sum`` (filtering.py:31-36)."""
    a = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty_like(a)
    _load().oracle_prefix_sum(_p64(a), _p64(out), a.size)
    return out


def filter_at(image, radii, weights, points) -> np.ndarray:
    """C restatement of ``filter_at`` (filtering.py:107-148), no validation."""
    a = np.ascontiguousarray(image, dtype=np.float64)
    h, w_ = a.shape
    r, w = _kernel_arrays(radii, weights)
    pts = np.asarray(points, dtype=np.int64).reshape(-1, 2)
    xs = np.ascontiguousarray(pts[:, 0])
    ys = np.ascontiguousarray(pts[:, 1])
    vals = np.empty(len(pts))
    cum = np.empty(h * w_)
    col = np.empty(h)
    colout = np.empty(h)
    if _load().oracle_filter_at(_p64(a), h, w_, _pi64(r), _p64(w), r.size, _pi64(xs), _pi64(ys), len(pts), _p64(vals),
                                _p64(cum), _p64(col), _p64(colout)):
        raise MemoryError("oracle_filter_at failed")
    return vals


_SRC_CODES = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.float32): 2, np.dtype(np.float64): 3}


def _image_view(image, channel):
    a = np.asarray(image)
    if a.dtype not in _SRC_CODES:
        a = a.astype(np.float64)
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    if a.ndim == 2:
        if channel:
            raise ValueError("channel given for a single-channel image")
        return a, a.shape[0], a.shape[1], 1, 0
    if a.ndim == 3:
        return a, a.shape[0], a.shape[1], a.shape[2], channel
    raise ValueError("need (H, W) or (H, W, C)")


def filter_columns(image, radii, weights, xs, channel: int = 0, threads: int = 8) -> np.ndarray:
    """Full output columns ``xs`` of separable_filter_2d (bit-identical to the
    reference: filter_at's arithmetic, filtering.py:126-148), O(width) memory.
    Returns an (H, len(xs)) float64 array."""
    a, h, w, c, ch = _image_view(image, channel)
    r, wt = _kernel_arrays(radii, weights)
    xs = np.ascontiguousarray(xs, dtype=np.int64)
    out = np.empty((len(xs), h))
    scratch = np.empty((len(xs), h))
    ptr = a.ctypes.data + ch * a.itemsize
    if _load().oracle_filter_columns(ptr, _SRC_CODES[a.dtype], h, w, c, _pi64(r), _p64(wt), r.size, _pi64(xs),
                                     len(xs), _p64(out), _p64(scratch), threads):
        raise MemoryError("oracle_filter_columns failed")
    return out.T.copy()


def filter_band(image, radii, weights, y0: int, y1: int, channel: int = 0, threads: int = 8) -> np.ndarray:
    """Output rows [y0, y1) of separable_filter_2d from input rows
    [y0-pmax-1, y1+pmax] only (float64; equal to the reference up to float64
    rounding of the shorter column prefix)."""
    a, h, w, c, ch = _image_view(image, channel)
    r, wt = _kernel_arrays(radii, weights)
    pmax = int(r[-1])
    out = np.empty((y1 - y0, w))
    n = min(h, y1 + pmax) - max(0, y0 - pmax - 1)
    scratch = np.empty((n, w))
    ptr = a.ctypes.data + ch * a.itemsize
    if _load().oracle_filter_band(ptr, _SRC_CODES[a.dtype], h, w, c, _pi64(r), _p64(wt), r.size, y0, y1, _p64(out),
                                  _p64(scratch), threads):
        raise MemoryError("oracle_filter_band failed")
    return out


# ---------------------------------------------------------------- numpy port
def np_filter_rows(arr: np.ndarray, radii, weights) -> np.ndarray:
    """numpy restatement of ``_filter_rows`` (filtering.py:48-64), same numpy ops."""
    m, n = arr.shape
    cum = np.cumsum(arr, axis=1)
    x = np.arange(n)
    out = np.zeros_like(arr)
    last = arr[:, -1:]
    first = arr[:, :1]
    for p, w in zip(radii, weights):
        hi_idx = x + p
        over = np.maximum(hi_idx - (n - 1), 0).astype(np.float64)
        hi = cum[:, np.minimum(hi_idx, n - 1)] + over * last
        lo_idx = x - p - 1
        under = np.minimum(lo_idx + 1, 0).astype(np.float64)
        lo = np.where(lo_idx < 0, under * first, cum[:, np.maximum(lo_idx, 0)])
        out += w * (hi - lo)
    return out


def np_separable_filter_2d(image, radii, weights, threads: int = 1) -> np.ndarray:
    """numpy restatement of ``separable_filter_2d``; ``threads`` > 1 splits each
    pass into row blocks over a thread pool (bit-identical, filtering.py:91-101)."""
    img = np.asarray(image, dtype=np.float64)
    r = np.asarray(radii, dtype=np.int64)
    w = np.asarray(weights, dtype=np.float64)

    def one_pass(arr):
        if threads <= 1 or arr.shape[0] < 64:
            return np_filter_rows(arr, r, w)
        blocks = np.array_split(np.arange(arr.shape[0]), threads)
        out = np.empty_like(arr)
        with ThreadPoolExecutor(max_workers=threads) as pool:
            for idx, res in zip(blocks, pool.map(lambda i: np_filter_rows(arr[i], r, w), blocks)):
                out[idx] = res
        return out

    rows = one_pass(img)
    return one_pass(rows.T).T

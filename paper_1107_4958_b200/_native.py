"""ctypes binding of ``libsliceblur_b200.so`` (include/sliceblur_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_1107_4958_b200.build``.  There is no fallback: if the shared
object is missing or cannot be loaded, every call raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os

LIB_NAME = "libsliceblur_b200.so"
LIB_PATH = os.environ.get("SB_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

SB_OK = 0
SB_ERR_INVALID_ARGUMENT = 1
SB_ERR_KERNEL_TOO_LARGE = 2
SB_ERR_NOT_UNIT_DC = 3
SB_ERR_CUDA = 4
SB_ERR_WORKSPACE = 5

SB_DTYPE_U8 = 0
SB_DTYPE_U16 = 1
SB_DTYPE_F32 = 2
SB_DTYPE_F64 = 3

SB_STATUS_RANGE = 1
SB_STATUS_HALF = 2
SB_MAX_K = 1024  # the templated sweep kernels take k <= 8; larger k runs the generic kernels
ABI_VERSION = 4

SB_PATH_AUTO = 0
SB_PATH_GENERIC = 1
SB_PATH_UNFUSED = 2
SB_PATH_U8_THREE_CTA = 3
SB_PATH_U8_ONE_BAND = 4
SB_PATH_FUSED_WIDE = 5
SB_PATH_U8_ROWTILE = 6
SB_PATH_U8_PAIRED = 7
SB_PATH_U8_TWO_BAND = 8

#: Every symbol include/sliceblur_b200.h declares (tests check the exports).
EXPORTED_SYMBOLS = (
    "sb_version",
    "sb_set_path_policy",
    "sb_last_error",
    "sb_check_kernel",
    "sb_separable_filter_2d_workspace_bytes",
    "sb_separable_filter_2d",
    "sb_separable_filter_2d_window",
    "sb_filter_rows_workspace_bytes",
    "sb_filter_rows",
    "sb_slice_filter_1d",
    "sb_prefix_sum_workspace_bytes",
    "sb_prefix_sum_f64",
    "sb_max_abs",
    "sb_filter_at_workspace_bytes",
    "sb_filter_at",
    "sb_exact_gaussian_workspace_bytes",
    "sb_exact_gaussian_2d",
    "sb_sum_sq_diff",
)


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing or failed to load."""


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_int = ctypes.c_int
_size = ctypes.c_size_t


def _declare(lib):
    lib.sb_version.argtypes = []
    lib.sb_version.restype = _int
    lib.sb_set_path_policy.argtypes = [_int]
    lib.sb_set_path_policy.restype = _int
    lib.sb_last_error.argtypes = []
    lib.sb_last_error.restype = ctypes.c_char_p
    lib.sb_check_kernel.argtypes = [_i64p, _f64p, _int, _i64]
    lib.sb_check_kernel.restype = _int
    lib.sb_separable_filter_2d_workspace_bytes.argtypes = [_int, _i64, _i64, _i64, _int, _i64p, _int]
    lib.sb_separable_filter_2d_workspace_bytes.restype = _size
    lib.sb_separable_filter_2d.argtypes = [
        _vp, _int, _i64, _i64, _i64, _int, _i64, _i64,  # src, dtype, batch, h, w, channels, img/row stride
        _vp, _i64, _i64,  # dst, img/row stride
        _i64p, _f64p, _int, ctypes.c_double,  # radii, weights, k, value_bound
        _vp, _size, _vp, _vp,  # workspace, bytes, status, stream
    ]
    lib.sb_separable_filter_2d.restype = _int
    lib.sb_separable_filter_2d_window.argtypes = [
        _vp, _int, _i64, _i64, _i64, _int, _i64, _i64,  # src, dtype, batch, h, w, channels, img/row stride
        _i64, _i64,  # row_begin, row_end
        _vp, _i64, _i64,  # dst, img/row stride
        _i64p, _f64p, _int, ctypes.c_double,
        _vp, _size, _vp, _vp,
    ]
    lib.sb_separable_filter_2d_window.restype = _int
    lib.sb_filter_rows_workspace_bytes.argtypes = [_int, _i64, _i64, _i64p, _int]
    lib.sb_filter_rows_workspace_bytes.restype = _size
    lib.sb_filter_rows.argtypes = [_vp, _int, _i64, _i64, _i64, _vp, _i64, _i64p, _f64p, _int, ctypes.c_double,
                                   _vp, _size, _vp, _vp]
    lib.sb_filter_rows.restype = _int
    lib.sb_slice_filter_1d.argtypes = [_vp, _int, _i64, _vp, _i64p, _f64p, _int, ctypes.c_double, _vp, _size, _vp,
                                       _vp]
    lib.sb_slice_filter_1d.restype = _int
    lib.sb_prefix_sum_workspace_bytes.argtypes = [_i64]
    lib.sb_prefix_sum_workspace_bytes.restype = _size
    lib.sb_prefix_sum_f64.argtypes = [_vp, _vp, _i64, _vp, _size, _vp]
    lib.sb_prefix_sum_f64.restype = _int
    lib.sb_max_abs.argtypes = [_vp, _int, _i64, _vp, _vp]
    lib.sb_max_abs.restype = _int
    lib.sb_filter_at_workspace_bytes.argtypes = [_i64, _i64]
    lib.sb_filter_at_workspace_bytes.restype = _size
    lib.sb_filter_at.argtypes = [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64p, _f64p, _int,
                                 ctypes.c_double, _vp, _size, _vp, _vp]
    lib.sb_filter_at.restype = _int
    lib.sb_exact_gaussian_workspace_bytes.argtypes = [_i64, _i64]
    lib.sb_exact_gaussian_workspace_bytes.restype = _size
    lib.sb_exact_gaussian_2d.argtypes = [_vp, _int, _i64, _i64, _i64, _vp, _int, _vp, _vp, _size, _vp]
    lib.sb_exact_gaussian_2d.restype = _int
    lib.sb_sum_sq_diff.argtypes = [_vp, _int, _vp, _int, _i64, _vp, _vp]
    lib.sb_sum_sq_diff.restype = _int


def load():
    """Load (once) and return the CDLL; raise NativeLibraryError if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_NAME} not found next to the package ({LIB_PATH}); build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)"
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the host
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        _declare(lib)
        if lib.sb_version() != ABI_VERSION:
            raise NativeLibraryError(f"{LIB_PATH} has ABI {lib.sb_version()}, this package needs {ABI_VERSION}; rebuild")
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().sb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


class path_policy:
    """Context manager forcing a path (SB_PATH_*) for the calls made on this thread.

    ``with path_policy(SB_PATH_GENERIC): ...`` runs the generic two-pass kernels; the
    tests use it to prove that every path gives bit-identical results.
    """

    def __init__(self, policy: int):
        self.policy = policy
        self.prev = None

    def __enter__(self):
        prev = load().sb_set_path_policy(self.policy)
        if prev < 0:
            raise ValueError(f"unknown path policy {self.policy}")
        self.prev = prev
        return self

    def __exit__(self, *exc):
        load().sb_set_path_policy(self.prev)
        return False

"""Drop-in GPU replacement of the reference filtering module.

Mirrors ``/root/reference/pkg/src/sliceblur/filtering.py``: same function
names, argument meaning and exceptions (``ValueError`` for bad shapes,
``KernelTooLargeError`` when a slice radius reaches an extent, ``ValueError``
for a non-unit-DC kernel).  Every call runs the sm_100a kernels of
``libsliceblur_b200.so`` through its C ABI; there is no CPU path.

Differences from the reference, by design:

* results are float32 (the reference returns float64); they agree with the
  reference within max-abs 1e-3 on a 0-255 scale (tests/test_gpu_parity.py);
* inputs may be numpy arrays (copied to the GPU and back) or CUDA
  ``torch.Tensor`` objects (filtered in place on the device, result returned
  as a CUDA tensor);
* float inputs are quantised to int32 fixed point with a quantum derived from
  ``value_bound`` (max |pixel|).  A pixel above the bound raises ``ValueError``,
  never a wrong answer.  When no bound is given, the previous image's measured
  maximum (per source dtype) is used as a guess and validated by the kernels'
  status word, which the call reads anyway (``SB_STATUS_RANGE`` clear and
  ``SB_STATUS_HALF`` set: the quantum is within one bit of the measured one);
  otherwise the maximum is measured on the device and the filter re-run.  So the
  reference signature ``separable_filter_2d(img, kern)`` costs no extra pass over
  the image in steady state.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .approx import SliceKernel

__all__ = [
    "KernelTooLargeError",
    "filter_at",
    "separable_filter_window",
    "filter_rows",
    "prefix_sum",
    "separable_filter_2d",
    "separable_filter_batch",
    "slice_filter_1d",
]

_DC_TOL = 1e-6


class KernelTooLargeError(ValueError):
    """A slice radius reaches or exceeds the filtered extent (filtering.py:27-28)."""


def _torch():
    import torch

    return torch


_DTYPE_CODES = {
    np.dtype(np.uint8): nat.SB_DTYPE_U8,
    np.dtype(np.uint16): nat.SB_DTYPE_U16,
    np.dtype(np.float32): nat.SB_DTYPE_F32,
    np.dtype(np.float64): nat.SB_DTYPE_F64,
}


# SliceKernel is immutable: its contiguous arrays, ctypes pointers and DC gain are
# computed once per kernel object (small images are host-bound otherwise).  The cache
# holds the kernel itself, so an id() is never reused while its entry exists.
_KERNEL_CACHE: "dict[int, tuple]" = {}
_KERNEL_CACHE_MAX = 64


def _kernel_info(kernel: SliceKernel):
    hit = _KERNEL_CACHE.get(id(kernel))
    if hit is not None and hit[0] is kernel:
        return hit
    radii = np.ascontiguousarray(kernel.radii, dtype=np.int64)
    weights = np.ascontiguousarray(kernel.weights, dtype=np.float64)
    info = (
        kernel,
        radii,
        weights,
        radii.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        weights.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        int(kernel.max_radius),
        float(kernel.dc_gain),
    )
    if len(_KERNEL_CACHE) >= _KERNEL_CACHE_MAX:
        _KERNEL_CACHE.clear()
    _KERNEL_CACHE[id(kernel)] = info
    return info


def _kernel_arrays(kernel: SliceKernel):
    return _kernel_info(kernel)[1:5]


def _raise_for(code: int):
    if code == nat.SB_OK:
        return
    msg = nat.last_error()
    if code == nat.SB_ERR_KERNEL_TOO_LARGE:
        raise KernelTooLargeError(msg)
    if code in (nat.SB_ERR_INVALID_ARGUMENT, nat.SB_ERR_NOT_UNIT_DC):
        raise ValueError(msg)
    raise RuntimeError(f"sliceblur_b200 error {code}: {msg}")


def _check_kernel(kernel: SliceKernel, n: int):
    """Mirror of filtering.py:39-45 (also enforced again inside the C ABI)."""
    info = _kernel_info(kernel)
    if info[5] >= n:
        raise KernelTooLargeError(f"slice radius {info[5]} does not fit extent {n}")
    if abs(info[6] - 1.0) > _DC_TOL:
        raise ValueError("kernel must have unit DC gain; call normalized()")
    if kernel.k > nat.SB_MAX_K:
        raise ValueError(f"at most {nat.SB_MAX_K} slices are supported")


class _Device:
    """Moves an input to the GPU (if needed) and remembers how to return the result."""

    _ready = False

    def __init__(self, data):
        torch = _torch()
        if not _Device._ready:
            if not torch.cuda.is_available():
                raise RuntimeError("sliceblur_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
            nat.load()
            _Device._ready = True
        self.torch = torch
        self.host_tensor = False
        if isinstance(data, torch.Tensor):
            self.from_numpy = False
            if data.is_cuda:
                t = data
            else:
                # host tensor (pinned for speed): H2D on the current stream
                self.host_tensor = True
                t = data.to(device="cuda", non_blocking=data.is_pinned())
        else:
            self.from_numpy = True
            arr = np.asarray(data)
            if arr.dtype not in _DTYPE_CODES:
                # the reference converts everything to float64 (filtering.py:84)
                arr = arr.astype(np.float64)
            t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        codes = {torch.uint8: nat.SB_DTYPE_U8, torch.float32: nat.SB_DTYPE_F32, torch.float64: nat.SB_DTYPE_F64}
        if hasattr(torch, "uint16"):
            codes[torch.uint16] = nat.SB_DTYPE_U16
        if t.dtype not in codes:
            t = t.to(torch.float64)
        self.tensor = t.contiguous()
        self.code = codes[self.tensor.dtype]
        self.stream = torch.cuda.current_stream().cuda_stream

    def measure_max(self) -> float:
        """max |pixel| on the device (one read of the input and a host sync)."""
        out = self.torch.zeros(1, dtype=self.torch.float64, device=self.tensor.device)
        _raise_for(nat.load().sb_max_abs(self.tensor.data_ptr(), self.code, self.tensor.numel(), out.data_ptr(),
                                          self.stream))
        bound = float(out.item())
        if not np.isfinite(bound):
            raise ValueError("input contains NaN or Inf; the fixed-point GPU path needs finite pixels")
        return bound

    def bound_for(self, given, check: bool):
        """(value_bound for the ABI, speculative?) - see the module docstring."""
        if self.code == nat.SB_DTYPE_U8:
            return 0.0, False  # exact integer path; bound implied by the dtype
        if given is not None:
            return float(given), False
        if self.code == nat.SB_DTYPE_U16:
            # exact samples either way; the measured maximum only refines the row-value quantum
            return max(1.0, self.measure_max()), False
        if check and self.code in _BOUND_GUESS:
            return _BOUND_GUESS[self.code], True
        bound = self.measure_max()
        _BOUND_GUESS[self.code] = bound
        return bound, False

    def run(self, launch, value_bound, check: bool, status=None):
        """launch(bound, status_ptr) -> ABI code; validates the status word once."""
        torch = self.torch
        own = status is None and check
        if own:
            status = torch.zeros(1, dtype=torch.int32, device=self.tensor.device)
        bound, spec = self.bound_for(value_bound, check)
        sp = status.data_ptr() if status is not None else None
        _raise_for(launch(bound, sp))
        if not own:
            return
        st = int(status.item())
        if spec and (st & nat.SB_STATUS_RANGE or not st & nat.SB_STATUS_HALF):
            # the guess does not fit this image: measure it and filter again
            bound = self.measure_max()
            _BOUND_GUESS[self.code] = bound
            status.zero_()
            _raise_for(launch(bound, sp))
            st = int(status.item())
        if st & nat.SB_STATUS_RANGE:
            raise ValueError("a pixel exceeds value_bound (or is not finite)")

    def finish(self, result, host_out=None):
        if host_out is not None:
            host_out.copy_(result.view(host_out.shape))
            return host_out
        if self.from_numpy:
            return result.cpu().numpy()
        if self.host_tensor:
            return result.cpu()
        return result


# last measured max |pixel| per float source dtype (the speculative bound, see above)
_BOUND_GUESS: "dict[int, float]" = {}


def _overlaps(a, b) -> bool:
    a0, b0 = a.data_ptr(), b.data_ptr()
    return a0 < b0 + b.numel() * b.element_size() and b0 < a0 + a.numel() * a.element_size()


def separable_filter_batch(images, kernel: SliceKernel, *, channels_last: bool = False, value_bound=None,
                           out=None, check: bool = True, _status=None):
    """Filter a batch of images: (B, H, W) or, with ``channels_last``,
    (B, H, W, C) / (H, W, C) with interleaved channels each filtered separately.

    The per-image arithmetic is ``separable_filter_2d``'s (filtering.py:76-104).
    Returns float32 of the input's shape (numpy in -> numpy out, CUDA tensor in
    -> CUDA tensor out, host tensor in -> host tensor out).  ``out`` may supply a
    preallocated contiguous float32 tensor of the input's shape: on the GPU it is
    written in place (it must not overlap the input), on the host (ideally pinned)
    the result is copied into it.
    """
    torch_mod = _torch()
    if (isinstance(images, torch_mod.Tensor) and not images.is_cuda and out is not None and not out.is_cuda
            and images.dim() >= 3 and (images.dim() == 4 or not channels_last) and images.shape[0] >= 4):
        return _pipelined_host_batch(images, kernel, channels_last, value_bound, out, check)
    dev = _Device(images)
    x = dev.tensor
    if channels_last:
        if x.dim() == 3:
            x = x.unsqueeze(0)
        if x.dim() != 4:
            raise ValueError("channels_last input must be (H, W, C) or (B, H, W, C)")
        b, h, w, c = x.shape
    else:
        if x.dim() == 2:
            x = x.unsqueeze(0)
        if x.dim() != 3:
            raise ValueError("need a (B, H, W) batch of 2D images")
        b, h, w = x.shape
        c = 1
    if min(b, h, w, c) < 1:
        raise ValueError("need a non-empty 2D image")
    _check_kernel(kernel, w)
    _check_kernel(kernel, h)
    torch = dev.torch
    host_out = None
    if out is not None:
        if out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != tuple(dev.tensor.shape):
            raise ValueError("out must be a contiguous float32 tensor of the input's shape")
        if out.is_cuda:
            if _overlaps(out, dev.tensor):
                raise ValueError("out must not overlap the input (the sweeps read rows other CTAs write)")
            result = out
        else:
            host_out = out  # D2H into the caller's (pinned) host buffer
            result = torch.empty(tuple(dev.tensor.shape), dtype=torch.float32, device=x.device)
    else:
        result = torch.empty(tuple(dev.tensor.shape), dtype=torch.float32, device=x.device)
    radii, weights, rp, wp = _kernel_arrays(kernel)
    lib = nat.load()
    ws_bytes = int(lib.sb_separable_filter_2d_workspace_bytes(dev.code, b, h, w, c, rp, kernel.k))
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device) if ws_bytes else None

    def launch(bound, status_ptr):
        return lib.sb_separable_filter_2d(
            x.data_ptr(), dev.code, b, h, w, c, h * w * c, w * c,
            result.data_ptr(), h * w * c, w * c,
            rp, wp, kernel.k, bound,
            workspace.data_ptr() if workspace is not None else None, ws_bytes, status_ptr, dev.stream)

    dev.run(launch, value_bound, check and _status is None, status=_status)
    return dev.finish(result, host_out)


def _pipelined_host_batch(images, kernel, channels_last, value_bound, out, check, chunks: int = 8):
    """Host batch -> host result with the PCIe copies overlapped with the kernel.

    The batch is cut into ``chunks`` image groups; group i is copied in on one
    stream while group i-1 is filtered on another and group i-2 copied out on a
    third (three device buffers rotate).  Every group runs with the same quanta as
    the one-shot call (float input: one bound for the whole batch - the caller's,
    the speculative guess, or the measured maximum), so the result is identical to
    it; the groups OR their status bits into one device word, read once at the end
    (no host sync between groups).
    """
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("sliceblur_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    if out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != tuple(images.shape):
        raise ValueError("out must be a contiguous float32 tensor of the input's shape")
    dev = torch.device("cuda", torch.cuda.current_device())
    code = {torch.float32: nat.SB_DTYPE_F32, torch.float64: nat.SB_DTYPE_F64}.get(images.dtype)
    is_float = code is not None
    spec = False
    bound = value_bound
    if is_float and bound is None:
        if check and code in _BOUND_GUESS:
            bound, spec = _BOUND_GUESS[code], True
        else:
            bound = float(images.abs().max())
            if not np.isfinite(bound):
                raise ValueError("input contains NaN or Inf; the fixed-point GPU path needs finite pixels")
            _BOUND_GUESS[code] = bound
    status = torch.zeros(1, dtype=torch.int32, device=dev) if check else None
    _run_pipeline(images, kernel, channels_last, bound, out, status, chunks)
    if not check:
        return out
    st = int(status.item())
    if spec and (st & nat.SB_STATUS_RANGE or not st & nat.SB_STATUS_HALF):
        bound = float(images.abs().max())
        if not np.isfinite(bound):
            raise ValueError("input contains NaN or Inf; the fixed-point GPU path needs finite pixels")
        _BOUND_GUESS[code] = bound
        status.zero_()
        _run_pipeline(images, kernel, channels_last, bound, out, status, chunks)
        st = int(status.item())
    if st & nat.SB_STATUS_RANGE:
        raise ValueError("a pixel exceeds value_bound (or is not finite)")
    return out


def _run_pipeline(images, kernel, channels_last, bound, out, status, chunks):
    torch = _torch()
    b = images.shape[0]
    chunks = max(1, min(chunks, b))
    bounds = [b * i // chunks for i in range(chunks + 1)]
    per = max(bounds[i + 1] - bounds[i] for i in range(chunks))
    dev = torch.device("cuda", torch.cuda.current_device())
    nbuf = 3
    xin = [torch.empty((per,) + tuple(images.shape[1:]), dtype=images.dtype, device=dev) for _ in range(nbuf)]
    yout = [torch.empty((per,) + tuple(images.shape[1:]), dtype=torch.float32, device=dev) for _ in range(nbuf)]
    s_in, s_run, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    main = torch.cuda.current_stream()
    for st in (s_in, s_run, s_out):
        st.wait_stream(main)
    done_run = [None] * nbuf
    done_out = [None] * nbuf
    for i in range(chunks):
        lo, hi = bounds[i], bounds[i + 1]
        n = hi - lo
        k = i % nbuf
        with torch.cuda.stream(s_in):
            if done_run[k] is not None:
                s_in.wait_event(done_run[k])  # input buffer k no longer read
            xin[k][:n].copy_(images[lo:hi], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
        with torch.cuda.stream(s_run):
            s_run.wait_event(ev_in)
            if done_out[k] is not None:
                s_run.wait_event(done_out[k])  # output buffer k copied out
            separable_filter_batch(xin[k][:n], kernel, channels_last=channels_last, value_bound=bound,
                                   out=yout[k][:n], check=status is not None, _status=status)
            done_run[k] = torch.cuda.Event()
            done_run[k].record(s_run)
        with torch.cuda.stream(s_out):
            s_out.wait_event(done_run[k])
            out[lo:hi].copy_(yout[k][:n], non_blocking=True)
            done_out[k] = torch.cuda.Event()
            done_out[k].record(s_out)
    for st in (s_in, s_run, s_out):
        main.wait_stream(st)
    s_out.synchronize()


def separable_filter_window(image, kernel: SliceKernel, row_begin: int, row_end: int, *, channels_last: bool = False,
                            value_bound=None, out=None, check: bool = True):
    """Rows [row_begin, row_end) of ``separable_filter_2d(image)`` (strip variant).

    ``image`` is (H, W) or, with ``channels_last``, (H, W, C).  Used by the
    row-strip partition (``distributed.filter_strip``): the image is a strip
    plus its neighbours' halo rows, and only the strip's own rows are output.
    Returns (row_end - row_begin, W[, C]) float32.
    """
    dev = _Device(image)
    x = dev.tensor
    if channels_last:
        if x.dim() != 3:
            raise ValueError("channels_last input must be (H, W, C)")
        h, w, c = x.shape
    else:
        if x.dim() != 2:
            raise ValueError("need a 2D image")
        h, w = x.shape
        c = 1
    if min(h, w, c) < 1:
        raise ValueError("need a non-empty 2D image")
    if not 0 <= row_begin < row_end <= h:
        raise ValueError("need 0 <= row_begin < row_end <= height")
    _check_kernel(kernel, w)
    _check_kernel(kernel, h)
    torch = dev.torch
    shape = (row_end - row_begin, w) + ((c,) if channels_last else ())
    result = out if out is not None else torch.empty(shape, dtype=torch.float32, device=x.device)
    if result.dtype != torch.float32 or not result.is_cuda or not result.is_contiguous() or tuple(result.shape) != shape:
        raise ValueError("out must be a contiguous float32 CUDA tensor of shape %r" % (shape,))
    if out is not None and _overlaps(result, x):
        raise ValueError("out must not overlap the input")
    radii, weights, rp, wp = _kernel_arrays(kernel)
    lib = nat.load()
    ws_bytes = int(lib.sb_separable_filter_2d_workspace_bytes(dev.code, 1, h, w, c, rp, kernel.k))
    workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)

    def launch(bound, status_ptr):
        return lib.sb_separable_filter_2d_window(
            x.data_ptr(), dev.code, 1, h, w, c, h * w * c, w * c, row_begin, row_end,
            result.data_ptr(), (row_end - row_begin) * w * c, w * c,
            rp, wp, kernel.k, bound, workspace.data_ptr(), ws_bytes, status_ptr, dev.stream)

    dev.run(launch, value_bound, check)
    return dev.finish(result)


def separable_filter_2d(image, kernel: SliceKernel, parallel: bool = False, *, value_bound=None, out=None,
                        check: bool = True):
    """Rows then columns, replicate boundary (filtering.py:76-104), on the GPU.

    ``parallel`` is accepted for signature compatibility and ignored (the GPU
    path is always parallel; the reference's results are identical either way).
    """
    del parallel
    if isinstance(image, np.ndarray) or not hasattr(image, "dim"):
        arr = np.asarray(image)
        if arr.ndim != 2:
            raise ValueError("need a 2D image")
    elif image.dim() != 2:
        raise ValueError("need a 2D image")
    return separable_filter_batch(image, kernel, value_bound=value_bound, out=out, check=check)


def filter_rows(arr, kernel: SliceKernel, *, value_bound=None, check: bool = True):
    """The row pass alone on every row of a 2D array (filtering.py:48-64)."""
    dev = _Device(arr)
    x = dev.tensor
    if x.dim() != 2 or x.shape[0] < 1 or x.shape[1] < 1:
        raise ValueError("need a non-empty 2D array")
    m, n = x.shape
    _check_kernel(kernel, n)
    return _rows_only(dev, x, m, n, kernel, value_bound, check, (m, n))


def _rows_only(dev, x, m, n, kernel, value_bound, check, shape):
    torch = dev.torch
    result = torch.empty(shape, dtype=torch.float32, device=x.device)
    radii, weights, rp, wp = _kernel_arrays(kernel)
    lib = nat.load()
    ws_bytes = int(lib.sb_filter_rows_workspace_bytes(dev.code, m, n, rp, kernel.k))
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device) if ws_bytes else None

    def launch(bound, status_ptr):
        return lib.sb_filter_rows(x.data_ptr(), dev.code, m, n, n, result.data_ptr(), n, rp, wp, kernel.k, bound,
                                  workspace.data_ptr() if workspace is not None else None, ws_bytes, status_ptr,
                                  dev.stream)

    dev.run(launch, value_bound, check)
    return dev.finish(result)


def slice_filter_1d(signal, kernel: SliceKernel, *, value_bound=None, check: bool = True):
    """Filter a 1D signal with a unit-gain slice kernel (filtering.py:67-73)."""
    dev = _Device(signal)
    x = dev.tensor
    if x.dim() != 1 or x.numel() < 1:
        raise ValueError("need a non-empty 1D signal")
    n = x.numel()
    _check_kernel(kernel, n)
    return _rows_only(dev, x, 1, n, kernel, value_bound, check, (n,))


def prefix_sum(values):
    """Inclusive float64 cumulative sum (filtering.py:31-36) on the GPU."""
    torch = _torch()
    if isinstance(values, torch.Tensor):
        t = values.to(device="cuda", dtype=torch.float64).contiguous()
        from_numpy = False
    else:
        arr = np.asarray(values, dtype=np.float64)
        if arr.ndim != 1 or arr.size < 1:
            raise ValueError("need a non-empty 1D signal")
        if not torch.cuda.is_available():
            raise RuntimeError("sliceblur_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
        t = torch.from_numpy(arr).cuda()
        from_numpy = True
    if t.dim() != 1 or t.numel() < 1:
        raise ValueError("need a non-empty 1D signal")
    lib = nat.load()
    n = t.numel()
    ws = int(lib.sb_prefix_sum_workspace_bytes(n))
    workspace = torch.empty(max(ws, 8), dtype=torch.uint8, device=t.device)
    out = torch.empty_like(t)
    _raise_for(lib.sb_prefix_sum_f64(t.data_ptr(), out.data_ptr(), n, workspace.data_ptr(), ws,
                                     torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy() if from_numpy else out


def filter_at(image, kernel: SliceKernel, points, *, value_bound=None, check: bool = True):
    """Evaluate the separable filter at selected (x, y) points only (filtering.py:107-148).

    The row pass runs only at the touched columns and the column pass only at
    the points (``sb_filter_at``); the values are bit-identical to the same
    pixels of ``separable_filter_2d`` on the GPU, as the reference's are to its
    own full filter.  Returns float32 values in point order (numpy for numpy
    input, a CUDA tensor for CUDA tensor input).
    """
    if isinstance(image, np.ndarray) or not hasattr(image, "dim"):
        if np.asarray(image).ndim != 2:
            raise ValueError("need a 2D image")
    elif image.dim() != 2:
        raise ValueError("need a 2D image")
    dev = _Device(image)
    x = dev.tensor
    h, w = x.shape
    if min(h, w) < 1:
        raise ValueError("need a non-empty 2D image")
    _check_kernel(kernel, w)
    _check_kernel(kernel, h)
    pts = [(int(px), int(py)) for px, py in points]
    for px, py in pts:
        if not (0 <= px < w and 0 <= py < h):
            raise ValueError(f"point ({px}, {py}) outside {w}x{h} image")
    torch = dev.torch
    if not pts:
        empty = torch.empty(0, dtype=torch.float32, device=x.device)
        return empty.cpu().numpy() if dev.from_numpy or dev.host_tensor else empty
    cols = sorted({px for px, _ in pts})
    index = {cx: i for i, cx in enumerate(cols)}
    cols_d = torch.tensor(cols, dtype=torch.int32).to(x.device)
    pt_col = torch.tensor([index[px] for px, _ in pts], dtype=torch.int32).to(x.device)
    pt_y = torch.tensor([py for _, py in pts], dtype=torch.int32).to(x.device)
    result = torch.empty(len(pts), dtype=torch.float32, device=x.device)
    radii, weights, rp, wp = _kernel_arrays(kernel)
    lib = nat.load()
    ws_bytes = int(lib.sb_filter_at_workspace_bytes(h, len(cols)))
    workspace = torch.empty(max(ws_bytes, 4), dtype=torch.uint8, device=x.device)

    def launch(bound, status_ptr):
        return lib.sb_filter_at(x.data_ptr(), dev.code, h, w, w, cols_d.data_ptr(), len(cols), pt_col.data_ptr(),
                                pt_y.data_ptr(), len(pts), result.data_ptr(), rp, wp, kernel.k, bound,
                                workspace.data_ptr(), ws_bytes, status_ptr, dev.stream)

    dev.run(launch, value_bound, check)
    return dev.finish(result)

"""GPU accuracy harness - mirror of the reference's ``oracle`` quality functions.

``/root/reference/pkg/src/sliceblur/oracle.py:58-102``: the dense truncated
Gaussian (``gaussian_taps``, ``exact_gaussian_2d``) the running-sum filter
approximates, and the ``mse`` / ``psnr`` metrics (images in [0, 1]).  Same
names, argument meaning and exceptions.  ``exact_gaussian_2d`` runs on the
device (``sb_exact_gaussian_2d``) with the reference's own fp64 operation
order, so it is bit-identical to it; ``mse`` reduces on the device
(``sb_sum_sq_diff``).  This is measurement tooling, not the hot path.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .filtering import _Device, _raise_for, _torch

__all__ = ["PSNR_INF", "exact_gaussian_2d", "gaussian_taps", "mse", "psnr"]

#: PSNR reported for identical images (MSE = 0), as the reference (oracle.py:20).
PSNR_INF = math.inf


def gaussian_taps(sigma: float) -> np.ndarray:
    """Dense 1D Gaussian with truncation radius ceil(pi * sigma), sum 1 (oracle.py:58-65)."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    r = math.ceil(math.pi * sigma)
    t = np.arange(-r, r + 1, dtype=np.float64)
    v = np.exp(-(t * t) / (2.0 * sigma * sigma))
    return v / v.sum()


def exact_gaussian_2d(image, sigma: float):
    """Reference Gaussian filtering: dense separable, replicate boundary (oracle.py:68-84).

    float64 result (numpy for numpy input, CUDA tensor for CUDA tensor input).
    """
    if isinstance(image, np.ndarray) or not hasattr(image, "dim"):
        if np.asarray(image).ndim != 2:
            raise ValueError("need a 2D image")
    elif image.dim() != 2:
        raise ValueError("need a 2D image")
    taps = gaussian_taps(sigma)
    dev = _Device(image)
    x = dev.tensor
    h, w = x.shape
    if min(h, w) < 1:
        raise ValueError("need a 2D image")
    torch = dev.torch
    taps_d = torch.from_numpy(taps).to(x.device)
    out = torch.empty((h, w), dtype=torch.float64, device=x.device)
    lib = nat.load()
    ws = int(lib.sb_exact_gaussian_workspace_bytes(h, w))
    work = torch.empty(max(ws, 8), dtype=torch.uint8, device=x.device)
    _raise_for(lib.sb_exact_gaussian_2d(x.data_ptr(), dev.code, h, w, w, taps_d.data_ptr(), taps.size,
                                        out.data_ptr(), work.data_ptr(), ws, dev.stream))
    if dev.from_numpy:
        return out.cpu().numpy()
    return out.cpu() if dev.host_tensor else out


def _as_device_float(a, torch):
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to("cuda")
    else:
        arr = np.asarray(a)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    return t.contiguous()


def mse(a, b) -> float:
    """Mean squared pixel difference (oracle.py:87-94)."""
    torch = _torch()
    shape_a = tuple(a.shape) if hasattr(a, "shape") else np.asarray(a).shape
    shape_b = tuple(b.shape) if hasattr(b, "shape") else np.asarray(b).shape
    if tuple(shape_a) != tuple(shape_b):
        raise ValueError("image dimensions must agree")
    if not torch.cuda.is_available():
        raise RuntimeError("sliceblur_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    ta, tb = _as_device_float(a, torch), _as_device_float(b, torch)
    n = ta.numel()
    if n == 0:
        return float("nan")  # numpy's mean of an empty array
    acc = torch.zeros(1, dtype=torch.float64, device=ta.device)
    code = {torch.float32: nat.SB_DTYPE_F32, torch.float64: nat.SB_DTYPE_F64}
    _raise_for(nat.load().sb_sum_sq_diff(ta.data_ptr(), code[ta.dtype], tb.data_ptr(), code[tb.dtype], n,
                                         acc.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return float(acc.item()) / n


def psnr(a, b) -> float:
    """-10 log10(MSE) for images in [0, 1]; PSNR_INF when identical (oracle.py:97-102)."""
    err = mse(a, b)
    if err == 0.0:
        return PSNR_INF
    return -10.0 * math.log10(err)

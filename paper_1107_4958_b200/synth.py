"""Seeded synthetic inputs for the BASELINE configurations.

The paper's 20-image Flickr corpus is not available and not needed; these
generators stand in for it with the shapes, sizes and value distributions
BASELINE.json names:

* ``one_over_f`` - a natural-like field: amplitude spectrum exactly ``1/|f|``
  on the ``fftfreq * N`` radial grid with DC = 0, phases i.i.d. U[0, 2*pi) from
  ``numpy.random.default_rng(seed)``, real field by ``irfft2`` of the
  half-plane spectrum (complex64 for sizes >= 8192^2), min-max rescaled to
  [0, 255], float32.  (The reference's own ``synth.make_image('one-over-f')``
  shapes Gaussian noise and rescales to [0, 1] (synth.py:28-38); parity is
  unaffected because the same array feeds both sides.)
* ``uniform_noise`` - i.i.d. U[0, 255) float32.
* ``impulse`` - 255 at the centre on zeros.
* ``to_u8`` - ``rint`` + clip to 0..255 (config 3).
"""

from __future__ import annotations

import numpy as np


def one_over_f(height: int, width: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    big = height * width >= 8192 * 8192
    cdtype = np.complex64 if big else np.complex128
    fdtype = np.float32 if big else np.float64
    fy = (np.fft.fftfreq(height) * height).astype(fdtype)[:, None]
    fx = (np.fft.rfftfreq(width) * width).astype(fdtype)[None, :]
    radius = np.hypot(fy, fx)
    amp = np.zeros_like(radius)
    np.divide(1.0, radius, out=amp, where=radius > 0)
    phase = rng.uniform(0.0, 2.0 * np.pi, size=radius.shape).astype(fdtype)
    spec = (amp * np.exp(1j * phase)).astype(cdtype)
    del amp, phase, radius
    field = np.fft.irfft2(spec, s=(height, width)).astype(np.float32)
    del spec
    lo, hi = float(field.min()), float(field.max())
    scale = np.float32(255.0 / (hi - lo)) if hi > lo else np.float32(0.0)
    field -= np.float32(lo)
    field *= scale
    np.clip(field, 0.0, 255.0, out=field)
    return field


def uniform_noise(height: int, width: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (rng.random((height, width), dtype=np.float32) * np.float32(255.0)).astype(np.float32)


def impulse(height: int, width: int) -> np.ndarray:
    img = np.zeros((height, width), dtype=np.float32)
    img[height // 2, width // 2] = 255.0
    return img


def to_u8(field: np.ndarray) -> np.ndarray:
    return np.clip(np.rint(field), 0, 255).astype(np.uint8)


def u8_batch(count: int, height: int, width: int, seed0: int = 1000) -> np.ndarray:
    """Config 3: ``count`` one-over-f images, seed ``seed0 + i``, rounded to u8."""
    out = np.empty((count, height, width), dtype=np.uint8)
    for i in range(count):
        out[i] = to_u8(one_over_f(height, width, seed0 + i))
    return out


def interleaved_rgb(height: int, width: int, seed0: int = 2000) -> np.ndarray:
    """Config 4: (H, W, 3) float32, channel c is one_over_f(seed0 + c)."""
    out = np.empty((height, width, 3), dtype=np.float32)
    for c in range(3):
        out[:, :, c] = one_over_f(height, width, seed0 + c)
    return out


def one_over_f_torch(height: int, width: int, seed: int, device="cuda"):
    """Same spectral definition as ``one_over_f``, generated on the GPU with
    ``torch.fft`` and a seeded ``torch.Generator`` (fast for 8192^2 .. 32768^2;
    deterministic per (seed, device type), different draws than numpy)."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    fy = (torch.fft.fftfreq(height, device=device) * height).float()[:, None]
    fx = (torch.fft.rfftfreq(width, device=device) * width).float()[None, :]
    radius = torch.hypot(fy, fx)
    amp = torch.where(radius > 0, 1.0 / torch.clamp(radius, min=1e-30), torch.zeros_like(radius))
    del radius
    phase = torch.rand(amp.shape, generator=gen, device=device, dtype=torch.float32) * (2.0 * np.pi)
    spec = torch.polar(amp, phase)
    del amp, phase
    field = torch.fft.irfft2(spec, s=(height, width))
    del spec
    lo, hi = field.min(), field.max()
    field = (field - lo) * (255.0 / (hi - lo))
    return field.clamp_(0.0, 255.0).contiguous()

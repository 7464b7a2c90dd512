"""Binary PGM (P5) I/O for the GPU filter CLI (reference: pgm.py:32-70).

``read_pgm`` / ``write_pgm`` keep the reference's semantics exactly: pixels map
to [0, 1] floats on read (``raw / maxval``), writes quantise with
``rint(clip(x, 0, 1) * maxval)``, 8-bit and 16-bit (big-endian) maxvals, and the
fixed header form ``P5\\n<w> <h>\\n<maxval>\\n`` so equal images give byte-identical
files.

``read_pgm_raw`` is the GPU path's reader: it returns the integer samples
(uint8, or native-endian uint16 for maxval > 255) so the device filters them
through the exact integer prefix (uint8 / uint16 -> int32), never through a
float conversion.  Filtering is linear, so ``filter(raw) / maxval`` equals the
reference's ``filter(raw / maxval)``.
"""

from __future__ import annotations

import re

import numpy as np


_HEADER = re.compile(rb"P5(?:\s|#[^\n]*\n)+(\d+)(?:\s|#[^\n]*\n)+(\d+)(?:\s|#[^\n]*\n)+(\d+)\s")


def read_pgm_raw(path) -> tuple[np.ndarray, int]:
    """Read a P5 file; returns (uint8 or uint16 samples of shape (h, w), maxval)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if not data.startswith(b"P5"):
        raise ValueError(f"{path}: not a binary PGM (P5) file")
    m = _HEADER.match(data)
    if m is None:
        raise ValueError(f"{path}: truncated PGM header")
    width, height, maxval = (int(v) for v in m.groups())
    if not 0 < maxval < 65536:
        raise ValueError(f"{path}: bad maxval {maxval}")
    wide = maxval > 255
    count = width * height
    nbytes = count * (2 if wide else 1)
    body = data[m.end():m.end() + nbytes]
    if len(body) != nbytes:
        raise ValueError(f"{path}: truncated pixel data")
    raw = np.frombuffer(body, dtype=">u2" if wide else np.uint8).reshape(height, width)
    return (raw.astype(np.uint16) if wide else raw.copy()), maxval  # native-endian samples for the device


def read_pgm(path) -> tuple[np.ndarray, int]:
    """Read a P5 file; returns (float64 image in [0, 1], maxval) like the reference."""
    raw, maxval = read_pgm_raw(path)
    return raw.astype(np.float64) / maxval, maxval


def quantize(image, maxval: int) -> np.ndarray:
    """``rint(clip(image, 0, 1) * maxval)`` in the file's sample type."""
    q = np.rint(np.clip(np.asarray(image, dtype=np.float64), 0.0, 1.0) * maxval)
    return q.astype(np.uint16 if maxval > 255 else np.uint8)


def write_samples(path, samples: np.ndarray, maxval: int):
    """Write already-quantised samples (uint8 / uint16) as P5."""
    if samples.ndim != 2:
        raise ValueError("need a 2D image")
    if not (0 < maxval < 65536):
        raise ValueError(f"bad maxval {maxval}")
    dtype = np.dtype(">u2") if maxval > 255 else np.dtype(np.uint8)
    h, w = samples.shape
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n%d\n" % (w, h, maxval))
        fh.write(samples.astype(dtype).tobytes())


def write_pgm(path, image, maxval: int = 255):
    """Quantise a [0, 1] float image and write it as P5 (reference pgm.py:57-70)."""
    image = np.asarray(image, dtype=np.float64)
    if image.ndim != 2:
        raise ValueError("need a 2D image")
    if not (0 < maxval < 65536):
        raise ValueError(f"bad maxval {maxval}")
    write_samples(path, quantize(image, maxval), maxval)

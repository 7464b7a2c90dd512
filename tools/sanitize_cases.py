"""Small cases of every warp-specialised / hand-synchronised kernel, for compute-sanitizer.

    compute-sanitizer --tool racecheck --kernel-name kns=sb:: python tools/sanitize_cases.py
    (one --tool per run: racecheck, synccheck, memcheck; see tools/sanitize.sh)

Each case runs one path (sb_set_path_policy) on a small input and checks the
result against the C oracle, so a sanitizer run also shows the kernels still
compute the right answer under instrumentation.  Shapes follow VERDICT r1 item
5: C1-sized, odd-sized, and the band-copy case (p_max 257).
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import approx as A  # noqa: E402
from paper_1107_4958_b200 import filtering as F  # noqa: E402

CASES = [
    # name, policy, dtype, (batch, h, w[, c]), k, sigma  -> kernels exercised
    ("u8 two-band fused (split 5)", nat.SB_PATH_AUTO, np.uint8, (3, 37, 150), 3, 4.0),
    ("u8 two-band fused, odd 61 images", nat.SB_PATH_AUTO, np.uint8, (61, 37, 150), 3, 3.0),
    ("u8 three-CTA fused (split 3)", nat.SB_PATH_U8_THREE_CTA, np.uint8, (5, 37, 150), 3, 3.0),
    ("u8 one-band fused", nat.SB_PATH_U8_ONE_BAND, np.uint8, (3, 37, 150), 3, 3.0),
    ("f32 fused (C1-sized)", nat.SB_PATH_AUTO, np.float32, (1, 512, 512), 3, 5.0),
    ("f32 fused, odd", nat.SB_PATH_AUTO, np.float32, (2, 131, 259), 4, 8.0),
    ("f32 stream rows + cols2, band copies (p_max 257)", nat.SB_PATH_AUTO, np.float32, (1, 700, 600), 4, 100.0),
    ("f32 stream rows + cols2, 2 channels, sigma 90", nat.SB_PATH_AUTO, np.float32, (1, 520, 530, 2), 5, 90.0),
    ("u16 tiled rows + cols kernels", nat.SB_PATH_UNFUSED, np.uint16, (2, 200, 150), 4, 8.0),
    ("f64 fused", nat.SB_PATH_AUTO, np.float64, (1, 96, 130), 5, 8.0),
    ("generic rows + cols", nat.SB_PATH_GENERIC, np.float32, (2, 150, 170, 3), 4, 20.0),
    ("f32 wide fused, band copies (p_max 257)", nat.SB_PATH_FUSED_WIDE, np.float32, (1, 700, 600), 4, 100.0),
    ("f32 wide fused, batch, odd width", nat.SB_PATH_FUSED_WIDE, np.float32, (3, 400, 517), 4, 40.0),
    ("u8 row-tile", nat.SB_PATH_U8_ROWTILE, np.uint8, (9, 300, 1000), 3, 10.0),
    ("u8 row-tile, tiny images", nat.SB_PATH_U8_ROWTILE, np.uint8, (61, 37, 150), 3, 3.0),
    # kernels of the last round-2 sessions
    ("u8 paired consumer warps", nat.SB_PATH_U8_PAIRED, np.uint8, (5, 37, 150), 3, 3.0),
    ("u8 paired consumer warps, odd 61 images", nat.SB_PATH_U8_PAIRED, np.uint8, (61, 37, 150), 3, 3.0),
    ("u8 paired consumer warps, 1000 wide", nat.SB_PATH_U8_PAIRED, np.uint8, (9, 300, 1000), 3, 10.0),
    ("f32 stream rows + cols2 split loader (ring only)", nat.SB_PATH_AUTO, np.float32, (1, 500, 600), 4, 40.0),
    ("f32 3 channels: stream_rows_mc + cols2 split loader", nat.SB_PATH_AUTO, np.float32, (2, 300, 388, 3), 4, 40.0),
    ("f32 4 channels, short images: stream_rows_mc", nat.SB_PATH_UNFUSED, np.float32, (5, 13, 388, 4), 3, 5.0),
]


def run_case(name, policy, dtype, shape, k, sigma):
    rng = np.random.default_rng(abs(hash(name)) % 2 ** 32)
    scale = 65535 if dtype == np.uint16 else 255
    x = (rng.random(shape) * scale).astype(dtype)
    kern = A.table_kernel(k, sigma)
    ch = shape[3] if len(shape) == 4 else 1
    bound = None if dtype in (np.uint8, np.uint16) else float(scale)
    with nat.path_policy(policy):
        got = F.separable_filter_batch(x, kern, channels_last=ch > 1, value_bound=bound)
    torch.cuda.synchronize()
    worst = 0.0
    for b in range(shape[0]):
        for c in range(ch):
            img = x[b, :, :, c] if ch > 1 else x[b]
            res = got[b, :, :, c] if ch > 1 else got[b]
            ref = O.separable_filter_2d(np.ascontiguousarray(img), kern.radii, kern.weights)
            worst = max(worst, float(np.abs(res - ref).max()) * 255.0 / scale)
    print(f"{name}: pmax {kern.max_radius} max_abs(0-255 scale) {worst:.2e}", flush=True)
    assert worst <= 1e-3, name


def main():
    torch.cuda.set_device(0)
    only = sys.argv[1:]
    for case in CASES:
        if only and not any(o in case[0] for o in only):
            continue
        run_case(*case)
    print("all cases ok", flush=True)


if __name__ == "__main__":
    main()

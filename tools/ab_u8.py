"""A/B of the uint8 sweeps on the C3 shape (256 x 1024^2, k3 sigma10) or a given batch:
SB_PATH_U8_ROWTILE (row-tile sweep) vs the automatic route (fused_kernel, two bands per
consumer turn) and the three-CTA variant; device time per call and bit-identity.

    python tools/ab_u8.py [BATCHxHxW:k:sigma ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import filtering, table_kernel  # noqa: E402


def timed(x, kern, out, iters):
    ts = []
    for i in range(iters + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        filtering.separable_filter_batch(x, kern, out=out, check=False)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    cases = sys.argv[1:] or ["256x1024x1024:3:10"]
    iters = int(os.environ.get("AB_ITERS", "9"))
    for c in cases:
        shape, k, sigma = c.split(":")
        n, h, w = map(int, shape.split("x"))
        kern = table_kernel(int(k), float(sigma))
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.randint(0, 256, (n, h, w), device="cuda", generator=g, dtype=torch.uint8)
        res = {}
        for name, pol in (("paired", nat.SB_PATH_U8_PAIRED), ("fused2", nat.SB_PATH_U8_TWO_BAND),
                          ("fused3", nat.SB_PATH_U8_THREE_CTA), ("rowtile", nat.SB_PATH_U8_ROWTILE)):
            out = torch.empty((n, h, w), device="cuda", dtype=torch.float32)
            with nat.path_policy(pol):
                t = timed(x, kern, out, iters)
            res[name] = (t, out)
        base = res["fused2"][1]
        line = "  ".join(f"{k_}: {t:.4f} ms ({n * h * w / t / 1e3:8.0f} Mpx/s) same={bool(torch.equal(o, base))}"
                         for k_, (t, o) in res.items())
        print(f"{c:20s} pmax={kern.max_radius:3d}  {line}", flush=True)


if __name__ == "__main__":
    main()

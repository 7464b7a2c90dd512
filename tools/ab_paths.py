"""A/B of the automatic route (or the policy AB_POLICY, e.g. 5 = SB_PATH_FUSED_WIDE) against the
two-launch path (SB_PATH_UNFUSED) on float32
images, on the GPU box: device time per call (CUDA events, median of --iters) and the
max-abs difference between the two results.

    python tools/ab_paths.py                 # the default case list
    python tools/ab_paths.py 8192x8192:4:64  # HxW:k:sigma ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import filtering, table_kernel  # noqa: E402

CASES = ["32768x32768:4:100", "16384x16384:4:100", "8192x8192:5:64", "8192x8192:4:32", "4096x4096:4:48",
         "2048x2048:4:32"]


def timed(x, kern, out, iters):
    ts = []
    for i in range(iters + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        filtering.separable_filter_batch(x, kern, value_bound=255.0, out=out, check=False)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    cases = sys.argv[1:] or CASES
    iters = int(os.environ.get("AB_ITERS", "5"))
    for c in cases:
        shape, k, sigma = c.split(":")
        h, w = map(int, shape.split("x"))
        kern = table_kernel(int(k), float(sigma))
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand((h, w), device="cuda", generator=g) * 255
        o1 = torch.empty_like(x)
        o2 = torch.empty_like(x)
        with nat.path_policy(int(os.environ.get("AB_POLICY", "0"))):
            t_auto = timed(x, kern, o1, iters)
        with nat.path_policy(nat.SB_PATH_UNFUSED):
            t_two = timed(x, kern, o2, iters)
        d = float((o1 - o2).abs().max())
        mpx = h * w / 1e6
        print(f"{c:22s} pmax={kern.max_radius:4d}  auto {t_auto:8.3f} ms ({1e3 * mpx / t_auto:9.0f} Mpx/s)  "
              f"two-launch {t_two:8.3f} ms ({1e3 * mpx / t_two:9.0f} Mpx/s)  max|diff| {d:.3e}", flush=True)
        del x, o1, o2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""Device time of the other reference entry points (GPU box): python tools/ab_api.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1107_4958_b200 import filtering, table_kernel  # noqa: E402


def timed(fn, iters=7):
    ts = []
    for i in range(iters + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    g = torch.Generator(device="cuda").manual_seed(1)
    for sigma in (8.0, 64.0):
        kern = table_kernel(4, sigma)
        for dt in (torch.float32, torch.float64, torch.uint8):
            sig = (torch.rand(1 << 24, device="cuda", generator=g) * 255).to(dt)
            img = (torch.rand((8192, 8192), device="cuda", generator=g) * 255).to(dt)
            vb = None if dt == torch.uint8 else 255.0
            t1 = timed(lambda: filtering.slice_filter_1d(sig, kern, value_bound=vb))
            t2 = timed(lambda: filtering.filter_rows(img, kern, value_bound=vb))
            t3 = timed(lambda: filtering.separable_filter_2d(img, kern, value_bound=vb))
            print(f"sigma {sigma:5.1f} pmax {kern.max_radius:3d} {str(dt).split('.')[-1]:8s} "
                  f"slice_filter_1d(2^24): {t1:.3f} ms  filter_rows(8192^2): {t2:.3f} ms  "
                  f"separable_filter_2d(8192^2): {t3:.3f} ms", flush=True)
    x = torch.rand(1 << 24, device="cuda", generator=g, dtype=torch.float64)
    print(f"prefix_sum(2^24 f64): {timed(lambda: filtering.prefix_sum(x)):.3f} ms")


if __name__ == "__main__":
    main()

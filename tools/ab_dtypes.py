"""Device time of the public call per source dtype on the same image (GPU box):

    python tools/ab_dtypes.py [HxW:k:sigma ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import filtering, table_kernel  # noqa: E402


def timed(x, kern, out, iters=7):
    cl = x.dim() == 4
    ts = []
    for i in range(iters + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        filtering.separable_filter_batch(x, kern, channels_last=cl,
                                         value_bound=None if x.dtype in (torch.uint8, torch.int16) else 255.0,
                                         out=out, check=False)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    nat.path_policy(int(os.environ.get("AB_POLICY", "0"))).__enter__()  # e.g. 2 = SB_PATH_UNFUSED
    cases = sys.argv[1:] or ["2048x2048:4:8", "4096x4096:4:30", "8192x8192:5:64"]
    for c in cases:
        shape, k, sigma = c.split(":")
        dims = list(map(int, shape.split("x")))  # HxW or HxWxC (interleaved channels)
        kern = table_kernel(int(k), float(sigma))
        g = torch.Generator(device="cuda").manual_seed(1)
        base = torch.rand((1, *dims), device="cuda", generator=g) * 255
        out = torch.empty((1, *dims), device="cuda", dtype=torch.float32)
        res = []
        for dt in (torch.float32, torch.float64, torch.uint8):
            x = base.to(dt)
            res.append(f"{str(dt).split('.')[-1]}: {timed(x, kern, out):.4f} ms")
        print(f"{c:18s} pmax={kern.max_radius:3d}  " + "  ".join(res), flush=True)


if __name__ == "__main__":
    main()

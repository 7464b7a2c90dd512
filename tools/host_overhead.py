"""Per-call host overhead of the public API on a small image (C1-size), on the GPU box.

    python tools/host_overhead.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1107_4958_b200 import filtering, table_kernel  # noqa: E402
from paper_1107_4958_b200 import _native as nat  # noqa: E402


def main():
    x = torch.rand(512, 512, device="cuda") * 255
    out = torch.empty_like(x)
    kern = table_kernel(3, 5.0)
    for _ in range(20):
        filtering.separable_filter_batch(x, kern, value_bound=255.0, out=out, check=False)
    torch.cuda.synchronize()
    n = 500
    t0 = time.perf_counter()
    for _ in range(n):
        filtering.separable_filter_batch(x, kern, value_bound=255.0, out=out, check=False)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e6
    # device time of the kernel alone: events around a burst with the host far ahead
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)  # let the host queue the burst before the GPU starts it
    e0.record()
    for _ in range(n):
        filtering.separable_filter_batch(x, kern, value_bound=255.0, out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / n * 1e3
    lib = nat.load()
    import ctypes
    import numpy as np
    rp = np.ascontiguousarray(kern.radii, np.int64)
    wp = np.ascontiguousarray(kern.weights, np.float64)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    args = (x.data_ptr(), nat.SB_DTYPE_F32, 1, 512, 512, 1, 512 * 512, 512, out.data_ptr(), 512 * 512, 512,
            rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), wp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            kern.k, 255.0, None, 0, status.data_ptr(), st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        lib.sb_separable_filter_2d(*args)
    torch.cuda.synchronize()
    cabi = (time.perf_counter() - t0) / n * 1e6
    print(f"public API wall {wall:.1f} us/call; C ABI alone {cabi:.1f} us/call; device {dev:.1f} us/call")


if __name__ == "__main__":
    main()

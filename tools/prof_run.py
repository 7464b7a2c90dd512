"""Small driver for ncu captures: runs one BASELINE config's filter `--iters` times.

    python tools/prof_run.py --config c3 --iters 3
    ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 1 \\
        -o gpurun_out/prof_c3 python tools/prof_run.py --config c3 --iters 3
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import filtering, table_kernel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(bench.CONFIGS))
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--policy", type=int, default=0, help="sb_set_path_policy value (SB_PATH_*)")
    args = ap.parse_args()
    nat.path_policy(args.policy).__enter__()
    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    x = bench.make_inputs(cfg, 1000, dev)
    out = torch.empty(x.shape, dtype=torch.float32, device=dev)
    kern = table_kernel(cfg["k"], cfg["sigma"])
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(args.iters):
        start.record()
        filtering.separable_filter_batch(x, kern, channels_last=cfg["channels"] > 1, value_bound=255.0, out=out,
                                         check=False)
        end.record()
        torch.cuda.synchronize()
        print(f"iter {i}: {start.elapsed_time(end):.3f} ms")


if __name__ == "__main__":
    main()

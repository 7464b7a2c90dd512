"""Race / bounds check without compute-sanitizer (closed on this pool).

    python tools/checked_run.py --save gpurun_out/chk              # production library
    SB_LIB_PATH=checked/libsliceblur_b200.so \
        python tools/checked_run.py --check gpurun_out/chk --reps 5  # SB_CHECKED library

--save writes every case of tools/sanitize_cases.py (each warp-specialised kernel,
every path policy, odd shapes, the band-copy case) as filtered by the production
library.  --check reruns them `reps` times with the checked library, whose kernels
trap on out-of-bounds shared-memory / TMEM indices and sleep pseudo-randomly at
every mbarrier arrive / wait, named barrier and bulk-store wait: every run must be
bit-identical to the production result (a missing wait or a buffer released early
would let some interleaving read stale or overwritten data) and a trap fails the
run.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import sanitize_cases as SC  # noqa: E402
from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import approx as A  # noqa: E402
from paper_1107_4958_b200 import filtering as F  # noqa: E402


def run(case):
    name, policy, dtype, shape, k, sigma = case
    rng = np.random.default_rng(sum(map(ord, name)))
    scale = 65535 if dtype == np.uint16 else 255
    x = (rng.random(shape) * scale).astype(dtype)
    kern = A.table_kernel(k, sigma)
    ch = shape[3] if len(shape) == 4 else 1
    bound = None if dtype in (np.uint8, np.uint16) else float(scale)
    with nat.path_policy(policy):
        got = F.separable_filter_batch(x, kern, channels_last=ch > 1, value_bound=bound)
    torch.cuda.synchronize()
    return got


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--save")
    ap.add_argument("--check")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    print("library:", nat.LIB_PATH, flush=True)
    bad = 0
    for i, case in enumerate(SC.CASES):
        if args.save:
            os.makedirs(args.save, exist_ok=True)
            np.save(os.path.join(args.save, f"case{i}.npy"), run(case))
            print(f"saved {case[0]}", flush=True)
            continue
        ref = np.load(os.path.join(args.check, f"case{i}.npy"))
        same = 0
        for _ in range(args.reps):
            same += int(np.array_equal(run(case), ref))
        ok = same == args.reps
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {case[0]}: {same}/{args.reps} runs bit-identical to the production library",
              flush=True)
    if args.check:
        print("checked run:", "all identical" if not bad else f"{bad} case(s) differ", flush=True)
        sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

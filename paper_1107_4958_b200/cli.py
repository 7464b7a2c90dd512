"""``sliceblur``-compatible command line on the B200 backend (reference: cli.py).

    python -m paper_1107_4958_b200.cli filter in.pgm out.pgm --sigma S [--k K | --params F] [--parallel]
    python -m paper_1107_4958_b200.cli optimize --k K [--model qf|l2] --params F [--samples N]
    python -m paper_1107_4958_b200.cli psnr a.pgm b.pgm

* ``filter`` (cli.py:71-76): the kernel is built on the host exactly as the
  reference builds it (Table II defaults or a parameter file, scaled to sigma,
  cli.py:61-68); the PGM's integer samples go to the device unconverted and
  are filtered through the exact uint8 / uint16 -> int32 prefix path of
  ``separable_filter_2d``; the result (in sample units, float32) is quantised
  as ``pgm.write_pgm`` does, ``rint(clip(x, 0, maxval))``.  Because the filter
  is linear this is the reference's ``rint(clip(filter(raw / maxval), 0, 1) *
  maxval)``; a sample can differ by one level only where the exact value lies
  within the GPU's ~1e-4 error of a rounding tie.
* ``optimize`` (cli.py:79-96): host box fitting (``approx.search_partitions``),
  bit-exact with the reference, written as a parameter file.
* ``psnr`` (cli.py:167-172): PSNR of two PGMs on the device (``quality.psnr``).

Errors map to exit status 2 with ``sliceblur: <message>`` on stderr, as the
reference's ``main`` does (cli.py:229-233).  ``bench`` and ``synth`` are not
part of the GPU path.
"""

from __future__ import annotations

import argparse
import math
import sys

import numpy as np

from . import approx, params, pgm


def scaled_kernel(k: int, sigma: float, params_path=None) -> approx.SliceKernel:
    """Kernel for ``filter``: a parameter file's partition or the Table II defaults, scaled to sigma."""
    if params_path is not None:
        loaded = params.load_params(params_path)
        base = approx.to_slices(loaded.partition, loaded.sigma0)
    else:
        base = approx.to_slices(*approx.table_defaults(k))
    return approx.scale_to_sigma(base, sigma)


def filter_samples(raw: np.ndarray, maxval: int, kernel: approx.SliceKernel) -> np.ndarray:
    """GPU filter of integer PGM samples, quantised back to the file's sample type."""
    from .filtering import separable_filter_2d

    out = separable_filter_2d(raw, kernel)  # float32, sample units, exact integer prefixes
    q = np.rint(np.clip(np.asarray(out, dtype=np.float64), 0.0, float(maxval)))
    return q.astype(np.uint16 if maxval > 255 else np.uint8)


def cmd_filter(args) -> int:
    kernel = scaled_kernel(args.k, args.sigma, args.params)
    raw, maxval = pgm.read_pgm_raw(args.input)
    pgm.write_samples(args.output, filter_samples(raw, maxval, kernel), maxval)
    return 0


def cmd_optimize(args) -> int:
    n = args.samples
    sigma0 = n / math.pi
    target = approx.sample_gaussian(sigma0, n)
    model = approx.build_autocorr(n - 1) if args.model == "qf" else approx.identity_model(n - 1)
    partition = approx.search_partitions(target, args.k, model)
    e2 = approx.quadratic_error(target, approx.partition_profile(partition, n), model)
    params.save_params(args.params, params.FilterParams(partition, sigma0, args.model, e2))
    return 0


def cmd_psnr(args) -> int:
    from .quality import psnr

    a, _ = pgm.read_pgm(args.image_a)
    b, _ = pgm.read_pgm(args.image_b)
    value = psnr(a, b)
    print("inf" if math.isinf(value) else repr(value))
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="sliceblur", description="Running-sum Gaussian filtering on B200")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("filter", help="blur a PGM image on the GPU")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--sigma", type=float, required=True)
    p.add_argument("--k", type=int, default=3, choices=(3, 4, 5))
    p.add_argument("--params", default=None, help="parameter file (overrides --k)")
    p.add_argument("--parallel", action="store_true", help="accepted for compatibility (the GPU path is parallel)")
    p.set_defaults(fn=cmd_filter)

    p = sub.add_parser("optimize", help="compute approximation parameters (host)")
    p.add_argument("--k", type=int, required=True, choices=range(1, 6))
    p.add_argument("--model", choices=("qf", "l2"), default="qf")
    p.add_argument("--params", required=True, help="output parameter file")
    p.add_argument("--samples", type=int, default=100, help="half-kernel samples")
    p.set_defaults(fn=cmd_optimize)

    p = sub.add_parser("psnr", help="PSNR between two PGM images")
    p.add_argument("image_a")
    p.add_argument("image_b")
    p.set_defaults(fn=cmd_psnr)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (OSError, ValueError) as exc:
        print(f"sliceblur: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

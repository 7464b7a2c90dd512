"""Golden fixtures for the CLI / PGM / parameter-file path, made by running the
reference package's own CLI HERE (never on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py

Writes into tests/golden/cli/:
* ``in8.pgm`` (61 x 47, maxval 255) and ``in16.pgm`` (53 x 40, maxval 4095):
  seeded 1/f fields (paper_1107_4958_b200.synth) quantised by the reference's
  ``write_pgm``;
* ``k4_l2.params``: ``sliceblur optimize --k 4 --model l2 --samples 40``;
* ``out8_s3_k3.pgm``, ``out16_s2.5_k5.pgm``, ``out8_s4_params.pgm``: the
  reference's ``sliceblur filter`` outputs for those inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(1, "/root/reference/pkg/src")

from paper_1107_4958_b200 import synth  # noqa: E402
from sliceblur import cli, pgm  # noqa: E402  (reference, read-only)


def main():
    os.makedirs(OUT, exist_ok=True)
    p = lambda name: os.path.join(OUT, name)  # noqa: E731
    pgm.write_pgm(p("in8.pgm"), synth.one_over_f(47, 61, 7) / 255.0, 255)
    pgm.write_pgm(p("in16.pgm"), synth.one_over_f(40, 53, 8) / 255.0, 4095)
    runs = [
        ["optimize", "--k", "4", "--model", "l2", "--samples", "40", "--params", p("k4_l2.params")],
        ["filter", p("in8.pgm"), p("out8_s3_k3.pgm"), "--sigma", "3", "--k", "3"],
        ["filter", p("in16.pgm"), p("out16_s2.5_k5.pgm"), "--sigma", "2.5", "--k", "5"],
        ["filter", p("in8.pgm"), p("out8_s4_params.pgm"), "--sigma", "4", "--params", p("k4_l2.params")],
    ]
    for argv in runs:
        rc = cli.main(argv)
        assert rc == 0, argv
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

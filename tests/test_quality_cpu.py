"""Host half of the accuracy harness (quality.py) against the reference's golden vectors."""

import os

import numpy as np
import pytest

from paper_1107_4958_b200 import quality as Q

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "quality_cases.npz")


def test_gaussian_taps_bit_exact_with_reference():
    z = np.load(GOLDEN)
    for name in sorted({k.split("/")[0] for k in z.files}):
        sigma = float(z[name + "/sigma"])
        taps = Q.gaussian_taps(sigma)
        np.testing.assert_array_equal(taps, z[name + "/taps"])
        assert taps.size == 2 * int(np.ceil(np.pi * sigma)) + 1


def test_gaussian_taps_rejects_nonpositive_sigma():
    with pytest.raises(ValueError):
        Q.gaussian_taps(0.0)
    with pytest.raises(ValueError):
        Q.gaussian_taps(-1.5)


def test_golden_metrics_are_consistent():
    # psnr = -10 log10(mse) as oracle.py:97-102 defines it
    z = np.load(GOLDEN)
    for name in sorted({k.split("/")[0] for k in z.files}):
        assert float(z[name + "/psnr"]) == pytest.approx(-10.0 * np.log10(float(z[name + "/mse"])), rel=1e-12)

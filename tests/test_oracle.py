"""Pin the oracle before trusting it.

The C restatement and the numpy port (oracle/) must reproduce the reference's
own outputs bit-for-bit on every golden case (tests/golden/filter_cases.npz,
made by running /root/reference via tests/golden/make_golden.py), and satisfy
the independent checks the reference's test-suite uses (dense-convolution
oracle, impulse box response, constant round trip; test_filtering.py:67-187).
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_1107_4958_b200 import approx as A


def _names(z):
    return sorted({k.split("/")[0] for k in z.files})


def test_golden_bit_exact(golden_cases):
    z = golden_cases
    checked = 0
    for name in _names(z):
        if name.startswith("prefix"):
            assert np.array_equal(O.prefix_sum(z[name + "/signal"]), z[name + "/out"])
        elif name == "filter_at":
            got = O.filter_at(z[name + "/image"], z[name + "/radii"], z[name + "/weights"], z[name + "/points"])
            assert np.array_equal(got, z[name + "/out"])
        elif name + "/signal" in z.files:
            sig = np.asarray(z[name + "/signal"], np.float64)[None, :]
            assert np.array_equal(O.filter_rows(sig, z[name + "/radii"], z[name + "/weights"])[0], z[name + "/out"])
        else:
            img, r, w = z[name + "/image"], z[name + "/radii"], z[name + "/weights"]
            ref = z[name + "/out"]
            assert np.array_equal(O.separable_filter_2d(img, r, w), ref), name
            assert np.array_equal(O.separable_filter_2d(img, r, w, threads=5), ref), name
            assert np.array_equal(O.np_separable_filter_2d(img, r, w), ref), name
            assert np.array_equal(O.np_separable_filter_2d(img, r, w, threads=4), ref), name
            xs = np.arange(img.shape[1])
            assert np.array_equal(O.filter_columns(img, r, w, xs, threads=3), ref), name
            y0, y1 = img.shape[0] // 3, img.shape[0] // 3 + 5
            assert np.abs(O.filter_band(img, r, w, y0, y1, threads=2) - ref[y0:y1]).max() <= 1e-9 * max(
                1.0, np.abs(ref).max())
        checked += 1
    assert checked == 25


def _dense_1d(sig, dense):
    r = dense.size // 2
    return np.convolve(np.pad(sig, r, mode="edge"), dense[::-1], mode="valid")


def test_dense_convolution_oracle():
    # test_filtering.py:89-97 style: random unit-gain kernels vs dense correlation
    rng = np.random.default_rng(9)
    for _ in range(40):
        n = int(rng.integers(8, 200))
        k = int(rng.integers(1, 6))
        max_p = min(n - 1, 40)
        k = min(k, max_p + 1)
        radii = np.sort(rng.choice(np.arange(max_p + 1), size=k, replace=False))
        kern = A.SliceKernel(radii, rng.uniform(0.1, 1.0, size=k)).normalized()
        sig = rng.random(n)
        fast = O.filter_rows(sig[None, :], kern.radii, kern.weights)[0]
        assert np.abs(fast - _dense_1d(sig, kern.dense())).max() <= 1e-10


def test_impulse_constant_2d():
    kern = A.SliceKernel((2,), (0.2,))
    sig = np.zeros(21)
    sig[10] = 1.0
    out = O.filter_rows(sig[None, :], kern.radii, kern.weights)[0]
    exp = np.zeros(21)
    exp[8:13] = 0.2
    np.testing.assert_allclose(out, exp, atol=1e-15)
    img = np.full((32, 48), 0.7)
    k3 = A.table_kernel(3, 2.0)
    np.testing.assert_allclose(O.separable_filter_2d(img, k3.radii, k3.weights), 0.7, atol=1e-12)


def test_outer_product_2d():
    rng = np.random.default_rng(23)
    img = rng.random((16, 16))
    kern = A.SliceKernel((1, 3), (0.08, 0.04)).normalized()
    d = kern.dense()
    k2 = np.outer(d, d)
    r = kern.max_radius
    pad = np.pad(img, r, mode="edge")
    exp = np.array([[np.sum(k2 * pad[y:y + 2 * r + 1, x:x + 2 * r + 1]) for x in range(16)] for y in range(16)])
    assert np.abs(O.separable_filter_2d(img, kern.radii, kern.weights) - exp).max() <= 1e-12


@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.float64])
def test_columns_and_bands_dtypes(dtype):
    rng = np.random.default_rng(5)
    img = (rng.random((90, 77)) * 255).astype(dtype)
    kern = A.table_kernel(4, 6.0)
    full = O.separable_filter_2d(img, kern.radii, kern.weights)
    cols = [0, 1, 38, 75, 76]
    assert np.array_equal(O.filter_columns(img, kern.radii, kern.weights, cols), full[:, cols])
    band = O.filter_band(img, kern.radii, kern.weights, 30, 60)
    assert np.abs(band - full[30:60]).max() <= 1e-9

"""GPU: the uint8 row-tile sweep (csrc/sweep_rowtile.cu, SB_PATH_U8_ROWTILE).

The row pass runs on thread-per-row warps that keep the row prefix in tensor memory; the
arithmetic is fused_kernel's, so the results must be bit-identical to the default uint8
path, and within the bar of the C oracle.  Shapes cover the persistent (row chunk, strip)
units: chunks split inside images, batches of tiny images, partial strips (W not a multiple
of 128), rows that are not 16-byte multiples (byte copies instead of cp.async), the border
replication of the first and last strip, and every k the templated kernel takes.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import approx as A  # noqa: E402
from paper_1107_4958_b200 import filtering as F  # noqa: E402

BAR = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("batch,h,w,k,sigma", [
    (24, 1024, 1024, 3, 10.0),  # the C3 image shape (a slice of the batch)
    (61, 37, 150, 3, 3.0),      # many tiny images, a partial second strip
    (7, 515, 300, 4, 8.0),
    (3, 200, 1001, 5, 6.0),     # W % 16 != 0: unaligned rows, byte copies
    (2, 333, 127, 1, 4.0),      # one partial strip, k = 1
    (5, 260, 520, 2, 9.0),
    (1, 64, 64, 3, 1.0),
])
def test_rowtile_bit_identical_to_fused_and_oracle(batch, h, w, k, sigma):
    rng = np.random.default_rng(batch * 7919 + h * 31 + w)
    if k in (3, 4, 5):
        kern = A.table_kernel(k, sigma)
    else:  # a user kernel: k boxes of radii up to ~sigma, weights normalised to unit DC
        radii = tuple(int(round(sigma * (i + 1) / k)) for i in range(k))
        kern = A.SliceKernel(radii, tuple(1.0 for _ in range(k))).normalized()
    if kern.max_radius >= min(h, w):
        pytest.skip("kernel larger than the image")
    x = torch.from_numpy(rng.integers(0, 256, size=(batch, h, w), dtype=np.uint8)).cuda()
    with nat.path_policy(nat.SB_PATH_U8_ROWTILE):
        a = F.separable_filter_batch(x, kern).cpu().numpy()
    b = F.separable_filter_batch(x, kern).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    xn = x.cpu().numpy()
    for i in sorted({0, batch // 2, batch - 1}):
        ref = O.separable_filter_2d(np.asarray(xn[i], np.float64), kern.radii, kern.weights)
        assert np.abs(a[i] - ref).max() <= BAR


def test_rowtile_row_window_and_fallback():
    """The row-window entry point (strip partition) through the row-tile sweep, and a radius
    past its TMEM budget falling back to the default sweep - both bit-identical."""
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.integers(0, 256, size=(900, 700), dtype=np.uint8)).cuda()
    for sigma in (10.0, 40.0):  # p_max 23 (row-tile) / 94 (past the row-tile budget)
        kern = A.table_kernel(3, sigma)
        with nat.path_policy(nat.SB_PATH_U8_ROWTILE):
            a = F.separable_filter_window(x, kern, 100, 650).cpu().numpy()
        b = F.separable_filter_window(x, kern, 100, 650).cpu().numpy()
        np.testing.assert_array_equal(a, b)

"""GPU: the one-launch wide fused sweep (csrc/sweep_wide.cu, SB_PATH_FUSED_WIDE).

float32 one-channel images with radii past the fused sweep (C2 sigma 32 .. C5 sigma 100):
bit-identical to the two-launch path (row plane + prefix-form column kernel) - the same
exact int32 prefixes, the same rounding of the row values and the same FFMA order - and
within the bar of the C oracle.  Shapes cover the persistent (row chunk, strip) units:
odd widths (element copies past the last 16-byte boundary), partial strips, batches
(segments split at image boundaries), row windows (strip partition), rows that are not
16-byte aligned (no bulk copies), and the band copies of trails older than the ring.
"""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_1107_4958_b200 import _native as nat  # noqa: E402
from paper_1107_4958_b200 import approx as A  # noqa: E402
from paper_1107_4958_b200 import filtering as F  # noqa: E402

BAR = 1e-3
THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _both(x, kern, **kw):
    with nat.path_policy(nat.SB_PATH_FUSED_WIDE):
        a = F.separable_filter_batch(x, kern, value_bound=255.0, **kw)
    with nat.path_policy(nat.SB_PATH_UNFUSED):
        b = F.separable_filter_batch(x, kern, value_bound=255.0, **kw)
    return a.cpu().numpy() if torch.is_tensor(a) else a, b.cpu().numpy() if torch.is_tensor(b) else b


@pytest.mark.parametrize("batch,h,w,k,sigma", [
    (1, 700, 300, 4, 100.0),    # p_max 257: band copies for the largest box, 3 strips
    (1, 1100, 250, 4, 75.0),    # tall, two strips (one partial)
    (3, 400, 260, 3, 40.0),     # a batch: units split at image boundaries
    (1, 2048, 2048, 4, 32.0),   # C2 sigma 32
    (2, 530, 517, 5, 64.0),     # odd width: element copies of the tail, partial last strip
    (1, 300, 1001, 4, 48.0),
])
def test_wide_bit_identical_to_two_launch_and_oracle(batch, h, w, k, sigma):
    rng = np.random.default_rng(batch * 1000 + h + w)
    kern = A.table_kernel(k, sigma)
    if kern.max_radius >= min(h, w):
        pytest.skip("kernel larger than the image")
    x = (rng.random((batch, h, w)) * 255).astype(np.float32)
    a, b = _both(torch.from_numpy(x).cuda(), kern)
    np.testing.assert_array_equal(a, b)
    for i in range(batch):
        if h * w <= 700 * 1100:
            ref = O.separable_filter_2d(np.asarray(x[i], np.float64), kern.radii, kern.weights)
        else:
            xs = np.array([0, 1, w // 2, w - 2, w - 1])
            ref = O.filter_columns(np.asarray(x[i], np.float64), kern.radii, kern.weights, xs, threads=THREADS)
            a_i = a[i][:, xs]
            assert np.abs(a_i - ref).max() <= BAR
            continue
        assert np.abs(a[i] - ref).max() <= BAR


def test_wide_unaligned_rows_and_windows():
    """Rows 4 bytes off 16-byte alignment (element copies instead of bulk copies) and the
    row-window entry point (strip partition) agree with the two-launch path bit for bit."""
    rng = np.random.default_rng(7)
    kern = A.table_kernel(4, 60.0)
    base = torch.from_numpy((rng.random((600, 421)) * 255).astype(np.float32)).cuda()
    x = base[:, 1:]  # row stride 421 floats: not a multiple of 16 bytes
    assert x.stride(0) * 4 % 16 != 0
    with nat.path_policy(nat.SB_PATH_FUSED_WIDE):
        a = F.separable_filter_2d(x, kern, value_bound=255.0).cpu().numpy()
        wa = F.separable_filter_window(base, kern, 150, 470, value_bound=255.0).cpu().numpy()
    with nat.path_policy(nat.SB_PATH_UNFUSED):
        b = F.separable_filter_2d(x, kern, value_bound=255.0).cpu().numpy()
        wb = F.separable_filter_window(base, kern, 150, 470, value_bound=255.0).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(wa, wb)
    ref = O.separable_filter_2d(np.asarray(x.cpu().numpy(), np.float64), kern.radii, kern.weights)
    assert np.abs(a - ref).max() <= BAR


def test_wide_range_status_and_needs_no_workspace():
    """A pixel above value_bound is reported (ValueError), as on every other path, and the
    wide sweep needs no workspace (the row values never leave the SM)."""
    kern = A.table_kernel(4, 50.0)
    x = torch.rand(400, 400, device="cuda") * 255
    x[123, 321] = 1000.0
    with nat.path_policy(nat.SB_PATH_FUSED_WIDE):
        with pytest.raises(ValueError):
            F.separable_filter_2d(x, kern, value_bound=255.0)
        radii = (ctypes.c_int64 * kern.k)(*[int(r) for r in kern.radii])
        assert nat.load().sb_separable_filter_2d_workspace_bytes(nat.SB_DTYPE_F32, 1, 400, 400, 1, radii, kern.k) == 0
    with nat.path_policy(nat.SB_PATH_UNFUSED):
        assert nat.load().sb_separable_filter_2d_workspace_bytes(nat.SB_DTYPE_F32, 1, 400, 400, 1, radii, kern.k) > 0

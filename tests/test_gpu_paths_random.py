"""GPU: randomized bit-identity of every path policy (SB_PATH_*) on the same inputs.

For random shapes, dtypes, channel counts, batches and user kernels (k = 1..8, p = 0,
negative weights, radii small and large), every policy that applies must give the SAME
bits as the default route: the generic kernels, the two-launch path, the
wide fused sweep (float32, one channel) and the row-tile sweep (uint8, one channel).  The
default route itself is checked against the C oracle.  SB_SWEEP_SEEDS sets the number of
cases (24 by default).
"""

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


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("seed", range(int(os.environ.get("SB_SWEEP_SEEDS", "24"))))
def test_every_policy_bit_identical(seed):
    rng = np.random.default_rng(77000 + seed)
    dtype = [np.uint8, np.float32, np.uint16, np.float64][seed % 4]
    h, w = int(rng.integers(2, 700)), int(rng.integers(2, 700))
    ch = int(rng.integers(2, 4)) if seed % 5 == 0 else 1
    batch = int(rng.integers(1, 4))
    reach = min(h, w) - 1
    k = int(min(rng.integers(1, 9), reach + 1))
    top = min(reach, [30, 300, 60][seed % 3])  # small radii (fused sweeps) or large (two launches / wide)
    pool = np.arange(0, top + 1)
    if pool.size < k:
        pool = np.arange(0, reach + 1)
    radii = np.sort(rng.choice(pool, size=k, replace=False))
    weights = rng.uniform(0.1, 1.0, size=k)
    if k > 1 and seed % 2:
        weights[int(rng.integers(k))] *= -0.3
    kern = A.SliceKernel(radii, weights).normalized()
    scale = {np.uint8: 255, np.uint16: 65535, np.float32: 255.0, np.float64: 1000.0}[dtype]
    bound = None if dtype in (np.uint8, np.uint16) else float(scale)
    shape = (batch, h, w, ch) if ch > 1 else (batch, h, w)
    x = torch.from_numpy((rng.random(shape) * scale).astype(dtype)).cuda()

    def run(policy):
        with nat.path_policy(policy):
            return F.separable_filter_batch(x, kern, channels_last=ch > 1, value_bound=bound).cpu().numpy()

    base = run(nat.SB_PATH_AUTO)
    policies = [nat.SB_PATH_GENERIC, nat.SB_PATH_UNFUSED, nat.SB_PATH_FUSED_WIDE, nat.SB_PATH_U8_ROWTILE,
                nat.SB_PATH_U8_PAIRED, nat.SB_PATH_U8_TWO_BAND]
    for pol in policies:
        np.testing.assert_array_equal(run(pol), base, err_msg=f"policy {pol} seed {seed}")
    gabs = float(np.sum(np.abs(kern.weights) * (2 * kern.radii + 1)))
    tol = BAR * float(scale) / 255.0 * max(1.0, gabs)
    xn = x.cpu().numpy()
    for bi in sorted({0, batch - 1}):
        for c in sorted({0, ch - 1}):
            img = xn[bi, :, :, c] if ch > 1 else xn[bi]
            ref = O.separable_filter_2d(np.ascontiguousarray(img), kern.radii, kern.weights)
            res = base[bi, :, :, c] if ch > 1 else base[bi]
            assert np.abs(res - ref).max() <= tol, (seed, h, w, dtype, ch, batch, kern)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SB_SWEEP_SEEDS", "24"))))
def test_windows_rows_and_wide_radii_bit_identical(seed):
    """The row-window entry point (strip partition), the row pass alone (filter_rows), very
    large radii (2 p_max + 1 > 2048: int64 generic kernels) and rows that are not 16-byte
    aligned (a column-sliced view), under every policy: the same bits as the default route."""
    rng = np.random.default_rng(88000 + seed)
    dtype = [np.float32, np.uint8, np.float64, np.uint16][seed % 4]
    wide = seed % 6 == 0
    h = int(rng.integers(2200, 2600)) if wide else int(rng.integers(3, 600))
    w = int(rng.integers(2200, 2600)) if wide and seed % 12 == 0 else int(rng.integers(3, 600))
    reach = min(h, w) - 1
    k = int(min(rng.integers(1, 9), reach + 1))
    top = reach if wide else min(reach, [40, 260, 120][seed % 3])
    lo = min(1030, top) if wide else 0
    pool = np.arange(lo, top + 1)
    if pool.size < k:
        pool = np.arange(0, reach + 1)
    radii = np.sort(rng.choice(pool, size=k, replace=False))
    kern = A.SliceKernel(radii, rng.uniform(0.1, 1.0, size=k)).normalized()
    scale = {np.uint8: 255, np.uint16: 65535, np.float32: 255.0, np.float64: 1000.0}[dtype]
    bound = None if dtype in (np.uint8, np.uint16) else float(scale)
    full = torch.from_numpy((rng.random((h, w + 1)) * scale).astype(dtype)).cuda()
    x = full[:, 1:] if seed % 2 else full[:, :w]  # odd seeds: rows 1 element off alignment
    r0 = int(rng.integers(0, h))
    r1 = int(rng.integers(r0 + 1, h + 1))

    def run(policy):
        with nat.path_policy(policy):
            a = F.separable_filter_window(x, kern, r0, r1, value_bound=bound).cpu().numpy()
            b = F.filter_rows(x, kern, value_bound=bound).cpu().numpy()
        return a, b

    base_w, base_r = run(nat.SB_PATH_AUTO)
    for pol in (nat.SB_PATH_GENERIC, nat.SB_PATH_UNFUSED, nat.SB_PATH_FUSED_WIDE, nat.SB_PATH_U8_ROWTILE,
                nat.SB_PATH_U8_PAIRED, nat.SB_PATH_U8_TWO_BAND):
        got_w, got_r = run(pol)
        np.testing.assert_array_equal(got_w, base_w, err_msg=f"window, policy {pol} seed {seed}")
        np.testing.assert_array_equal(got_r, base_r, err_msg=f"rows, policy {pol} seed {seed}")
    if not wide:  # the oracle on a band of the window (full columns at this size are cheap)
        xn = np.ascontiguousarray(x.cpu().numpy(), np.float64)
        ref = O.filter_band(xn, kern.radii, kern.weights, r0, r1, threads=8)
        tol = BAR * float(scale) / 255.0
        assert np.abs(base_w - ref).max() <= tol, (seed, h, w, dtype, kern)

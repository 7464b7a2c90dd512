"""Host-side caches of the GPU wrapper (no device needed).

``filtering._kernel_info`` caches a SliceKernel's contiguous arrays, ctypes
pointers and DC gain per kernel object; an id() reused by a new kernel must
never return the old entry, and the checks must match the reference's
``_check_kernel`` (filtering.py:39-45).
"""

import gc

import numpy as np
import pytest

from paper_1107_4958_b200 import filtering as F
from paper_1107_4958_b200 import table_kernel
from paper_1107_4958_b200.approx import SliceKernel


def test_kernel_info_matches_kernel_and_survives_id_reuse():
    for k, sigma in [(3, 5.0), (4, 8.0), (5, 64.0)] * 20:
        kern = table_kernel(k, sigma)
        info = F._kernel_info(kern)
        assert info[0] is kern
        assert np.array_equal(info[1], kern.radii) and np.array_equal(info[2], kern.weights)
        assert info[1].dtype == np.int64 and info[2].dtype == np.float64
        assert info[3].contents.value == int(kern.radii[0]) and info[4].contents.value == float(kern.weights[0])
        assert info[5] == kern.max_radius and info[6] == kern.dc_gain
        del kern, info
        gc.collect()
    assert len(F._KERNEL_CACHE) <= F._KERNEL_CACHE_MAX


def test_check_kernel_uses_cached_values_like_the_reference():
    kern = table_kernel(3, 5.0)
    F._check_kernel(kern, kern.max_radius + 1)
    with pytest.raises(F.KernelTooLargeError):
        F._check_kernel(kern, kern.max_radius)
    bad = SliceKernel(np.array([1, 2]), np.array([0.1, 0.1]))  # dc gain 0.8
    with pytest.raises(ValueError, match="unit DC"):
        F._check_kernel(bad, 100)

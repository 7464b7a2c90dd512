"""Host box model: bit-exact with the reference (golden vectors from running it).

Pins: tests/golden/box_params.json (tests/golden/make_golden.py ran the
reference's table_defaults/to_slices/scale_to_sigma/search_partitions).  The
property tests restate the reference's own test_approx.py checks
(test_approx.py:277-282, 320-348, 355-368).
"""

import math

import numpy as np
import pytest

from paper_1107_4958_b200 import approx as A


def _hex(values):
    return [float(v).hex() for v in np.asarray(values, dtype=np.float64).ravel()]


def test_sigma0_bits(box_params):
    assert float(A.SIGMA0).hex() == box_params["sigma0"]


def test_table_kernels_bit_exact(box_params):
    bases = {}
    for k in (3, 4, 5):
        part, s0 = A.table_defaults(k)
        bases[k] = A.to_slices(part, s0)
        assert _hex(bases[k].weights) == box_params[f"base_weights_k{k}"]
    n = 0
    for entry in box_params["table"]:
        sigma = float.fromhex(entry["sigma"])
        if entry.get("degenerate"):
            with pytest.raises(A.DegenerateScaleError):
                A.scale_to_sigma(bases[entry["k"]], sigma)
            continue
        kern = A.scale_to_sigma(bases[entry["k"]], sigma)
        assert kern.radii.tolist() == entry["radii"], (entry["k"], sigma)
        assert _hex(kern.weights) == entry["weights"], (entry["k"], sigma)
        assert float(kern.dc_gain).hex() == entry["dc_gain"]
        n += 1
    assert n > 300


@pytest.mark.parametrize(
    "k,sigma,radii",
    [
        (3, 5.0, [3, 7, 11]),
        (4, 2.0, [1, 2, 3, 5]),
        (4, 8.0, [4, 9, 14, 20]),
        (4, 32.0, [19, 37, 56, 82]),
        (3, 10.0, [7, 14, 23]),
        (5, 64.0, [32, 60, 88, 122, 170]),
        (4, 100.0, [59, 116, 175, 257]),
    ],
)
def test_baseline_config_radii(k, sigma, radii):
    # SURVEY.md Appendix A (reference run): all distinct, no merges
    assert A.table_kernel(k, sigma).radii.tolist() == radii


def test_appendix_a_weights_hex():
    kern = A.table_kernel(4, 100.0)
    assert _hex(kern.weights) == [
        "0x1.39b6304982f01p-10", "0x1.5fafd31c48041p-10", "0x1.fe3c8311d2596p-11", "0x1.9e285c91e2f0ap-12"]
    kern = A.table_kernel(3, 10.0)
    assert _hex(kern.weights) == ["0x1.fde2d14fb7bb8p-7", "0x1.0088e7ccdfb4dp-6", "0x1.b3c62df426aefp-8"]


def test_sample_gaussian_and_autocorr_bits(box_params):
    target = A.sample_gaussian(100.0 / math.pi, 100)
    assert _hex(target.values) == box_params["sample_gaussian_100"]
    assert _hex(A.build_autocorr(99).phi) == box_params["autocorr_r99_phi"]


def test_search_partitions_match_reference(box_params):
    target = A.sample_gaussian(100.0 / math.pi, 100)
    models = {"qf": A.build_autocorr(99), "l2": A.identity_model(99)}
    for entry in box_params["fitted"]:
        part = A.search_partitions(target, entry["k"], models[entry["model"]])
        assert part.breakpoints.tolist() == entry["breakpoints"], entry["model"]
        # LAPACK-dependent bits: exact on the same numpy build, else 1e-12
        np.testing.assert_allclose(part.constants, [float.fromhex(h) for h in entry["constants"]], rtol=0,
                                   atol=1e-12)
        e2 = A.quadratic_error(target, A.partition_profile(part, 100), models[entry["model"]])
        assert e2 == pytest.approx(float.fromhex(entry["e2"]), rel=1e-9, abs=1e-18)
        kern = A.to_slices(part, 100.0 / math.pi)
        for s_hex, scaled in entry["scaled"].items():
            if scaled is None:
                with pytest.raises(A.DegenerateScaleError):
                    A.scale_to_sigma(kern, float.fromhex(s_hex))
                continue
            sk = A.scale_to_sigma(kern, float.fromhex(s_hex))
            assert sk.radii.tolist() == scaled["radii"]


class TestReferenceProperties:
    def test_table_values(self):
        p3, s0 = A.table_defaults(3)
        assert s0 == pytest.approx(100.0 / math.pi, rel=1e-15)
        assert p3.breakpoints.tolist() == [23, 46, 76]
        np.testing.assert_allclose(p3.constants, (0.9495, 0.5502, 0.1618))

    @pytest.mark.parametrize("k", [1, 2, 6])
    def test_table_bad_k(self, k):
        with pytest.raises(ValueError):
            A.table_defaults(k)

    def test_builtin_k3_weights(self):
        part, _ = A.table_defaults(3)
        np.testing.assert_allclose(A.to_slices(part).weights, (0.3993, 0.3884, 0.1618), atol=1e-12)

    def test_half_sigma_radii(self):
        part, s0 = A.table_defaults(3)
        assert A.scale_to_sigma(A.to_slices(part, s0), s0 / 2.0).radii.tolist() == [11, 23, 38]

    def test_unit_dc(self):
        part, s0 = A.table_defaults(3)
        for sigma in (0.8, 2.0, 7.7, 31.0, 80.0):
            assert abs(A.scale_to_sigma(A.to_slices(part, s0), sigma).dc_gain - 1.0) <= 1e-12

    def test_collision_and_degenerate(self):
        base = A.to_slices(A.Partition((4, 5), (1.0, 0.5)), 10.0)
        scaled = A.scale_to_sigma(base, 3.0)
        assert scaled.radii.tolist() == [1]
        assert abs(scaled.dc_gain - 1.0) <= 1e-12
        with pytest.raises(A.DegenerateScaleError):
            A.scale_to_sigma(base, 0.5)
        with pytest.raises(ValueError):
            A.scale_to_sigma(base, 0.0)

    def test_slice_kernel_validation(self):
        with pytest.raises(ValueError):
            A.SliceKernel((), ())
        with pytest.raises(ValueError):
            A.SliceKernel((3, 3), (0.1, 0.1))
        with pytest.raises(ValueError):
            A.SliceKernel((-1,), (1.0,))
        with pytest.raises(ValueError):
            A.SliceKernel((1, 2), (1.0,))
        k = A.SliceKernel((0, 2), (0.5, 0.1))
        assert k.k == 2 and k.max_radius == 2
        with pytest.raises(AttributeError):
            k.radii = np.array([1])

    def test_dense_reconstruction(self):
        rng = np.random.default_rng(11)
        for _ in range(20):
            k = int(rng.integers(1, 6))
            bp = np.sort(rng.choice(np.arange(1, 40), size=k, replace=False))
            part = A.Partition(bp, rng.standard_normal(k))
            kern = A.to_slices(part)
            prof = A.partition_profile(part, int(bp[-1]) + 1)
            dense = kern.dense()
            c = kern.max_radius
            for t in range(int(bp[-1]) + 1):
                assert dense[c + t] == pytest.approx(prof[t], abs=1e-12)
                assert dense[c - t] == pytest.approx(prof[t], abs=1e-12)

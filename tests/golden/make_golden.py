"""Generate the golden fixtures by running the reference package itself.

Run HERE (the build container), never on the GPU box:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``sliceblur`` read-only from ``/root/reference/pkg/src`` and writes

* ``box_params.json`` - table-default kernels ``scale_to_sigma(to_slices(
  *table_defaults(k)), sigma)`` for k in {3,4,5} over a sigma sweep, the fitted
  partitions ``search_partitions(sample_gaussian(100/pi, 100), k, model)`` for
  k in 1..5 and model in {qf, l2}, and ``build_autocorr(99)``'s Phi, all as
  ``float.hex`` so the host restatement can be checked bit-for-bit;
* ``filter_cases.npz`` - small seeded inputs with the reference's own
  ``separable_filter_2d`` / ``slice_filter_1d`` / ``prefix_sum`` /
  ``filter_at`` outputs (float64), covering the edge cases its tests cover:
  impulse, constant, both boundary clamps at once (2p+1 > n), p = 0,
  negative slice weights, non-square and odd shapes, f32 and u8 inputs.

The committed fixtures are the parity anchor on the GPU box, where
``/root/reference`` does not exist.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def _load_reference():
    sys.path.insert(0, REF_SRC)
    import sliceblur  # noqa: E402  (reference package, read-only)

    return sliceblur


def _hex(values):
    return [float(v).hex() for v in np.asarray(values, dtype=np.float64).ravel()]


def box_params(sb):
    out = {"table": [], "fitted": [], "autocorr_r99_phi": None, "sigma0": float(sb.approx.SIGMA0).hex()}
    rng = np.random.default_rng(20261019)
    sigmas = sorted(
        set(
            [0.8, 1.0, 1.5, 2.0, 3.0, 4.0, 5.0, 7.7, 8.0, 10.0, 16.0, 20.0, 31.0, 32.0, 50.0, 64.0, 80.0, 100.0,
             100.0 / math.pi, 50.0 / math.pi, 128.0, 200.0]
            + [float(s) for s in rng.uniform(0.5, 150.0, size=120)]
        )
    )
    for k in (3, 4, 5):
        part, s0 = sb.table_defaults(k)
        base = sb.to_slices(part, s0)
        out["base_weights_k%d" % k] = _hex(base.weights)
        for s in sigmas:
            try:
                kern = sb.scale_to_sigma(base, s)
            except sb.DegenerateScaleError:
                out["table"].append({"k": k, "sigma": float(s).hex(), "degenerate": True})
                continue
            out["table"].append(
                {
                    "k": k,
                    "sigma": float(s).hex(),
                    "radii": kern.radii.tolist(),
                    "weights": _hex(kern.weights),
                    "dc_gain": float(kern.dc_gain).hex(),
                }
            )
    target = sb.sample_gaussian(100.0 / math.pi, 100)
    out["sample_gaussian_100"] = _hex(target.values)
    models = {"qf": sb.build_autocorr(99), "l2": sb.approx.identity_model(99)}
    out["autocorr_r99_phi"] = _hex(models["qf"].phi)
    for name, model in models.items():
        for k in range(1, 6):
            part = sb.search_partitions(target, k, model)
            e2 = sb.quadratic_error(target, sb.approx.partition_profile(part, 100), model)
            kern = sb.to_slices(part, 100.0 / math.pi)
            scaled = {}
            for s in (2.0, 8.0, 10.0, 32.0, 64.0, 100.0):
                try:
                    sk = sb.scale_to_sigma(kern, s)
                    scaled[float(s).hex()] = {"radii": sk.radii.tolist(), "weights": _hex(sk.weights)}
                except sb.DegenerateScaleError:
                    scaled[float(s).hex()] = None
            out["fitted"].append(
                {
                    "model": name,
                    "k": k,
                    "breakpoints": part.breakpoints.tolist(),
                    "constants": _hex(part.constants),
                    "e2": float(e2).hex(),
                    "scaled": scaled,
                }
            )
    return out


def filter_cases(sb):
    """Seeded small cases; every array the reference produced is stored float64."""
    SliceKernel = sb.SliceKernel
    rng = np.random.default_rng(1107_4958)
    cases = {}

    def table(k, s):
        part, s0 = sb.table_defaults(k)
        return sb.scale_to_sigma(sb.to_slices(part, s0), s)

    def put2d(name, img, kern):
        cases[f"{name}/image"] = np.asarray(img)
        cases[f"{name}/radii"] = np.asarray(kern.radii, dtype=np.int64)
        cases[f"{name}/weights"] = np.asarray(kern.weights, dtype=np.float64)
        cases[f"{name}/out"] = sb.separable_filter_2d(img, kern)

    def put1d(name, sig, kern):
        cases[f"{name}/signal"] = np.asarray(sig)
        cases[f"{name}/radii"] = np.asarray(kern.radii, dtype=np.int64)
        cases[f"{name}/weights"] = np.asarray(kern.weights, dtype=np.float64)
        cases[f"{name}/out"] = sb.slice_filter_1d(sig, kern)

    # 2D, float64 inputs in [0,1) like the reference tests
    put2d("rand64_k3s4", rng.random((64, 64)), table(3, 4.0))
    put2d("rand37x53_k4s3", rng.random((37, 53)), table(4, 3.0))
    put2d("rand48x72_k3s3", rng.random((48, 72)), table(3, 3.0))
    # both clamps at once: 2p+1 > n in both dimensions
    put2d("tiny11x13_both_clamps", rng.random((11, 13)), SliceKernel((0, 4, 9), (0.5, -0.1, 0.2)).normalized())
    # radius 0 slice and negative weights
    put2d("p0_negw_20x31", rng.random((20, 31)), SliceKernel((0, 2, 5), (0.9, -0.3, 0.4)).normalized())
    imp = np.zeros((64, 64))
    imp[32, 32] = 1.0
    put2d("impulse64_k4s4", imp, table(4, 4.0))
    put2d("const32x48_k3s2", np.full((32, 48), 0.7), table(3, 2.0))
    # f32 inputs on the 0..255 scale (the BASELINE configs' scale)
    f32 = (rng.random((96, 128)) * 255.0).astype(np.float32)
    put2d("f32_96x128_k3s5", f32, table(3, 5.0))
    put2d("f32_96x128_k4s8", f32, table(4, 8.0))
    f32b = (rng.random((200, 180)) * 255.0).astype(np.float32)
    put2d("f32_200x180_k5s20", f32b, table(5, 20.0))
    put2d("f32_200x180_k4s32", f32b, table(4, 32.0))
    # u8 inputs
    u8 = rng.integers(0, 256, size=(64, 80), dtype=np.uint8)
    put2d("u8_64x80_k3s10", u8, table(3, 10.0))
    u8b = rng.integers(0, 256, size=(130, 70), dtype=np.uint8)
    put2d("u8_130x70_k4s8", u8b, table(4, 8.0))
    # random kernels in the style of the reference test suite (test_filtering.py:22-29)
    for i in range(6):
        h, w = int(rng.integers(8, 90)), int(rng.integers(8, 90))
        kk = int(rng.integers(1, 6))
        max_p = min(min(h, w) - 1, 40)
        kk = min(kk, max_p + 1)
        radii = np.sort(rng.choice(np.arange(max_p + 1), size=kk, replace=False))
        weights = rng.uniform(0.1, 1.0, size=kk)
        put2d(f"randkern{i}_{h}x{w}", rng.random((h, w)) * 255.0, SliceKernel(radii, weights).normalized())
    # 1D
    put1d("sig64_k3s4", rng.random(64), table(3, 4.0))
    put1d("sig21_impulse_box", np.eye(1, 21, 10)[0], SliceKernel((2,), (0.2,)))
    put1d("sig300_k5s30", rng.random(300) * 255.0, table(5, 30.0))
    put1d("sig7_both_clamps", rng.random(7), SliceKernel((1, 6), (0.05, 0.06)).normalized())
    # prefix sum
    sig = rng.standard_normal(100)
    cases["prefix100/signal"] = sig
    cases["prefix100/out"] = sb.prefix_sum(sig)
    # filter_at
    img = rng.random((24, 30))
    kern = table(3, 2.0)
    pts = np.array([(int(rng.integers(30)), int(rng.integers(24))) for _ in range(40)], dtype=np.int64)
    cases["filter_at/image"] = img
    cases["filter_at/radii"] = kern.radii
    cases["filter_at/weights"] = kern.weights
    cases["filter_at/points"] = pts
    cases["filter_at/out"] = sb.filter_at(img, kern, [tuple(p) for p in pts])
    return cases


def quality_cases(sb):
    """The reference's accuracy harness (oracle.py:58-102): dense truncated Gaussian
    taps, ``exact_gaussian_2d``, and ``mse`` / ``psnr`` of the running-sum filter
    against it, on small seeded images."""
    import sliceblur.oracle as so  # noqa: E402

    rng = np.random.default_rng(20261)
    cases = {}
    for name, shape, sigma, k in [("q40x50_s1p5", (40, 50), 1.5, 3), ("q64x80_s3", (64, 80), 3.0, 4),
                                  ("q120x96_s8", (120, 96), 8.0, 5)]:
        img = rng.random(shape)
        kern = sb.table_kernel(k, sigma) if hasattr(sb, "table_kernel") else None
        if kern is None:
            from sliceblur.approx import scale_to_sigma, table_defaults, to_slices
            kern = scale_to_sigma(to_slices(*table_defaults(k)), sigma)
        exact = so.exact_gaussian_2d(img, sigma)
        fast = sb.separable_filter_2d(img, kern)
        cases[name + "/image"] = img
        cases[name + "/sigma"] = np.float64(sigma)
        cases[name + "/taps"] = so.gaussian_taps(sigma)
        cases[name + "/exact"] = exact
        cases[name + "/radii"] = kern.radii
        cases[name + "/weights"] = kern.weights
        cases[name + "/mse"] = np.float64(so.mse(fast, exact))
        cases[name + "/psnr"] = np.float64(so.psnr(fast, exact))
    return cases


def main():
    sb = _load_reference()
    np.savez_compressed(os.path.join(HERE, "quality_cases.npz"), **quality_cases(sb))
    params = box_params(sb)
    with open(os.path.join(HERE, "box_params.json"), "w") as fh:
        json.dump(params, fh, indent=1, sort_keys=True)
    cases = filter_cases(sb)
    np.savez_compressed(os.path.join(HERE, "filter_cases.npz"), **cases)
    print(f"wrote {len(params['table'])} table kernels, {len(params['fitted'])} fitted partitions, "
          f"{len([c for c in cases if c.endswith('/out')])} filter cases")


if __name__ == "__main__":
    main()

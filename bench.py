"""Benchmark of the B200 running-sum Gaussian filter (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Workload (default c3 = BASELINE.json configs[2]): a batch of 256 uint8
1024x1024 one-over-f images filtered with sigma=10, K=3 table boxes
(radii 7/14/23) into float32 - the config the metric's 1/2/4/8-GPU scaling is
quoted on.  Multi-GPU: one process per GPU (torchrun), every rank filters its
own 256-image batch (weak scaling, no data-path collective); timing is CUDA
events on the launching stream, max over ranks.

* ``value``    - Mpixels/s over all ranks with inputs resident in HBM
                 (inputs 268 MB + outputs 1 GB per rank > 126 MB L2, so no flush
                 is needed between steps);
* ``e2e``      - the same metric through the public API
                 (``separable_filter_batch``) from pinned host memory, H2D of
                 the input and D2H of the filtered images inside the timed region;
* ``roofline`` - algorithmic bytes (1 read of the input + 1 write of the output
                 per pixel) per launch / CUDA-event launch time vs the measured
                 HBM copy peak (MEASURED_PEAKS.json);
* ``cpu_baseline`` - the reference algorithm's numpy port (oracle/), all host
                 cores, on a bounded sample, rank 0 at N=1.

``--impl reference`` times that CPU implementation alone (rank 0; other ranks
exit 0) on the same metric/config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Gaussian-filtered Mpixels/s"
UNIT = "Mpx/s"

CONFIGS = {
    "c1": dict(batch=1, h=512, w=512, channels=1, dtype="f32", k=3, sigma=5.0,
               desc="BASELINE configs[0]: 512x512 f32 1/f, sigma=5, K=3"),
    "c2": dict(batch=1, h=2048, w=2048, channels=1, dtype="f32", k=4, sigma=8.0,
               desc="BASELINE configs[1]: 2048x2048 f32 1/f, sigma=8, K=4"),
    "c3": dict(batch=256, h=1024, w=1024, channels=1, dtype="u8", k=3, sigma=10.0,
               desc="BASELINE configs[2]: 256 x 1024x1024 u8 1/f -> f32, sigma=10, K=3"),
    "c4": dict(batch=1, h=8192, w=8192, channels=3, dtype="f32", k=5, sigma=64.0,
               desc="BASELINE configs[3]: 8192x8192x3 interleaved f32 1/f, sigma=64, K=5"),
    "c5": dict(batch=1, h=32768, w=32768, channels=1, dtype="f32", k=4, sigma=100.0,
               desc="BASELINE configs[4]: 32768x32768 f32 1/f, sigma=100, K=4"),
}


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _traffic_from_profiles(config_name):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config_name)
    except (OSError, ValueError):
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 100 ms in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "samples": len(sm),
                "reasons": sorted(reasons)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_inputs(cfg, seed_base, device):
    """Seeded synthetic inputs of the config, generated on the GPU (torch.fft)."""
    import torch

    from paper_1107_4958_b200 import synth

    if cfg["dtype"] == "u8":
        out = torch.empty((cfg["batch"], cfg["h"], cfg["w"]), dtype=torch.uint8, device=device)
        for i in range(cfg["batch"]):
            out[i] = synth.one_over_f_torch(cfg["h"], cfg["w"], seed_base + i, device=device).round_().to(torch.uint8)
        return out
    if cfg["channels"] == 1:
        return synth.one_over_f_torch(cfg["h"], cfg["w"], seed_base, device=device).unsqueeze(0)
    out = torch.empty((1, cfg["h"], cfg["w"], cfg["channels"]), dtype=torch.float32, device=device)
    for c in range(cfg["channels"]):
        out[0, :, :, c] = synth.one_over_f_torch(cfg["h"], cfg["w"], seed_base + c, device=device)
    return out


def cpu_reference_rate(cfg, sample_px_target: float, threads: int, reps: int = 1):
    """Time the reference algorithm's numpy port (oracle/) on a bounded sample.

    Returns (Mpx/s, sample description).  Uses a thread pool over row blocks
    like the reference's parallel=True (filtering.py:91-101), on ``threads`` cores.
    """
    from oracle import oracle
    from paper_1107_4958_b200 import synth, table_kernel

    kern = table_kernel(cfg["k"], cfg["sigma"])
    side_h, side_w = cfg["h"], cfg["w"]
    if cfg["dtype"] == "u8":
        img = synth.to_u8(synth.one_over_f(side_h, side_w, 1000))
    else:
        # a sample band of the full-width image keeps the per-row cost of the real size
        rows = int(max(2 * kern.max_radius + 2, min(side_h, sample_px_target // side_w)))
        img = synth.one_over_f(rows, side_w, 42)
    per_image = img.size
    n_img = max(1, int(sample_px_target // per_image)) if cfg["dtype"] == "u8" else 1
    channels = cfg["channels"]
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for _i in range(n_img):
            for _c in range(channels):
                oracle.np_separable_filter_2d(img, kern.radii, kern.weights, threads=threads)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    px = n_img * per_image  # per-pixel metric counts each RGB pixel once (all channels)
    desc = (f"{n_img} x {img.shape[0]}x{img.shape[1]} {cfg['dtype']} image(s) x {channels} channel(s), "
            f"numpy port of filtering.py, {threads}-thread pool over row blocks, median of {reps}")
    return px / t / 1e6, desc


def run_reference(args, cfg):
    world, rank, _ = _dist()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    sample = 4 * 1024 * 1024 if cfg["dtype"] == "u8" else 2 * 1024 * 1024
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, sample / 4, threads)
    rates = []
    t0 = time.perf_counter()
    desc = ""
    for _ in range(args.steps):
        r, desc = cpu_reference_rate(cfg, sample, threads)
        rates.append(r)
    elapsed = time.perf_counter() - t0
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * elapsed / max(1, args.steps), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"]},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_1107_4958_b200 import _native as nat
    from paper_1107_4958_b200 import distributed as D
    from paper_1107_4958_b200 import filtering, table_kernel

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    kern = table_kernel(cfg["k"], cfg["sigma"])
    channels_last = cfg["channels"] > 1
    bound = 255.0
    # config 5 on several GPUs: one image partitioned into row strips with a halo
    # exchange; every other config: each rank filters its own batch (no collective)
    strips = args.config == "c5" and world > 1
    if strips:
        full = make_inputs(cfg, 42, device)[0]  # same seed on every rank: identical image
        r0, r1 = D.shard_range(cfg["h"], rank, world)
        x = full[r0:r1].contiguous()
        del full
        out = torch.empty(x.shape, dtype=torch.float32, device=device)
        px_per_rank = (r1 - r0) * cfg["w"]
        px_total = cfg["h"] * cfg["w"]
        scaling = "strong"
    else:
        x = make_inputs(cfg, 1000 + rank * 100000 if cfg["dtype"] == "u8" else 42 + rank, device)
        out = torch.empty(x.shape, dtype=torch.float32, device=device)
        px_per_rank = cfg["batch"] * cfg["h"] * cfg["w"]
        px_total = px_per_rank * world
        scaling = "weak"
    in_bytes = x.numel() * x.element_size()
    out_bytes = out.numel() * out.element_size()
    alg_bytes = in_bytes + out_bytes

    lib = nat.load()
    rp = np.ascontiguousarray(kern.radii, np.int64)
    dcode = nat.SB_DTYPE_U8 if cfg["dtype"] == "u8" else nat.SB_DTYPE_F32
    ws = lib.sb_separable_filter_2d_workspace_bytes(dcode, cfg["batch"], cfg["h"], cfg["w"], cfg["channels"],
                                                    rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), kern.k)
    launches_per_step = 1 if ws == 0 else 2
    if strips:
        def step():
            D.filter_strip(x, kern, channels_last=channels_last, value_bound=bound, out=out)
    else:
        def step():
            filtering.separable_filter_batch(x, kern, channels_last=channels_last, value_bound=bound, out=out,
                                             check=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    # keep the GPU loaded ~1 s more (untimed) so the clock sampler sees the load
    t_end = time.time() + max(0.0, 1.2 - ms / 1e3)
    while time.time() < t_end:
        step()
        torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_max = D.max_over_ranks(ms, device=device)
    ms_per_step = ms_max / args.steps
    value = px_total * args.steps / (ms_max / 1e3) / 1e6

    # e2e through the public API from pinned host memory (H2D of the inputs and
    # D2H of the filtered images inside the timed region)
    x_host = x.cpu().pin_memory()
    out_host = torch.empty(out.shape, dtype=torch.float32).pin_memory()
    if strips:
        def e2e_step():
            res = D.filter_strip(x_host.to(device, non_blocking=True), kern, channels_last=channels_last,
                                 value_bound=bound, out=out)
            out_host.copy_(res)
    else:
        def e2e_step():
            filtering.separable_filter_batch(x_host, kern, channels_last=channels_last, value_bound=bound,
                                             out=out_host, check=False)
    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e_ms = D.max_over_ranks((time.perf_counter() - t0) * 1e3, device=device)
    e_value = px_total * e_steps / (e_ms / 1e3) / 1e6

    # sampled parity on this rank's output (not timed)
    from oracle import oracle

    threads = len(os.sched_getaffinity(0))
    if strips:
        max_abs = rmse = None  # checked by tests/test_gpu_parity.py::test_row_window_strips_match_full_image
    else:
        xs = x[0].cpu().numpy()
        got = out[0].cpu().numpy()
        if channels_last:
            xs, got = xs[:, :, 0], got[:, :, 0]
        if cfg["h"] * cfg["w"] <= 4096 * 4096:
            ref = oracle.separable_filter_2d(xs, kern.radii, kern.weights, threads=threads)
            diff = got.astype(np.float64) - ref
        else:
            cols = np.array([0, cfg["w"] // 2, cfg["w"] - 1])
            ref = oracle.filter_columns(xs, kern.radii, kern.weights, cols, threads=threads)
            diff = got[:, cols].astype(np.float64) - ref
        max_abs = float(np.abs(diff).max())
        rmse = float(np.sqrt(np.mean(diff * diff)))
    # quality of the K-box approximation against the dense truncated Gaussian (the
    # reference's own harness, oracle.py:58-102, here on the GPU), image 0, [0, 1] scale
    quality = None
    if not strips and cfg["h"] * cfg["w"] <= 8192 * 8192:
        from paper_1107_4958_b200 import quality as Q

        img0 = x[0] if not channels_last else x[0][:, :, 0].contiguous()
        fast0 = out[0] if not channels_last else out[0][:, :, 0].contiguous()
        exact0 = Q.exact_gaussian_2d(img0, cfg["sigma"])
        quality = {"psnr_db_vs_exact_gaussian": round(Q.psnr(fast0 / 255.0, exact0 / 255.0), 3),
                   "scope": "rank-0 image 0 (channel 0), values / 255, exact = dense Gaussian r = ceil(pi*sigma)"}

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, desc = cpu_reference_rate(cfg, 4 * 1024 * 1024 if cfg["dtype"] == "u8" else 2 * 1024 * 1024, threads)
        cpu = {"value": round(rate, 3), "unit": UNIT, "cores": threads, "kind": "port", "sample": desc}
    peak, peak_kind = _peaks()
    # algorithmic bytes of a step (one read of every input pixel, one write of every output
    # pixel) over the CUDA-event step time; for the two-launch path the pair is the unit
    achieved = alg_bytes / (ms_per_step / 1e3) / 1e9
    traffic = _traffic_from_profiles(args.config)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "source_dtype": cfg["dtype"], "output_dtype": "f32",
                   "per_gpu_images": cfg["batch"] if not strips else None,
                   "global_images": cfg["batch"] * world if not strips else 1,
                   "height": cfg["h"], "width": cfg["w"], "channels": cfg["channels"], "k": cfg["k"],
                   "sigma": cfg["sigma"], "radii": kern.radii.tolist(),
                   "parallelism": (f"row strips x{world} + NCCL halo exchange" if strips
                                   else f"dp{world} (image batch sharded, no collective)"),
                   "l2": ("inputs+outputs per step exceed the 126 MB L2; no flush" if alg_bytes > 2 * 126e6 else
                          "working set fits the 126 MB L2 (parity-size config)")},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_step": alg_bytes,
                     "kernel": "fused_kernel (one launch per step)" if ws == 0 else
                               "stream_rows_kernel + cols2_kernel (two launches per step, timed together)"},
        "e2e": {"value": round(e_value, 1), "unit": UNIT, "h2d_bytes_per_step": int(in_bytes),
                "d2h_bytes_per_step": int(out_bytes)},
        "gpu_launches": int(args.steps * launches_per_step),
        "parity": {"max_abs": max_abs, "rmse": rmse, "scope": "rank-0 image 0 vs C oracle"},
        "quality": quality,
        "clocks": clocks,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()

"""World-size 2/3 CPU (gloo) tests of the multi-GPU plumbing.

The row-strip partition (config 5) must reproduce the full-image result: each
rank receives its neighbours' halo rows over point-to-point sends into its
persistent [halo | strip | halo] buffer, and ``distributed.filter_strip`` -
with the interior/edge-band overlap and without - must equal the same rows of
the whole-image reference.  Here the row-window filter is the float64 oracle's
band filter (the row-window semantics of sb_separable_filter_2d_window), so the
decomposition itself is what is tested; the GPU kernels are exercised by
tests/test_gpu_parity.py.  Batch sharding (config 3) must cover every image once,
and a strip thinner than the halo must make every rank raise (no P2P hang).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1107_4958_b200 import distributed as D
from paper_1107_4958_b200.approx import table_kernel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_window(img, kern, r0, r1, out=None, **_):
    from oracle import oracle as O

    res = O.filter_band(np.ascontiguousarray(img.numpy(), np.float64), kern.radii, kern.weights, r0, r1, threads=2)
    out.copy_(torch.from_numpy(res.astype(np.float32)))
    return out


def _worker(rank, world, port, h, w, sigma, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        rng = np.random.default_rng(123)
        img = (rng.random((h, w)) * 255).astype(np.float32)
        kern = table_kernel(k, sigma)
        r0, r1 = D.shard_range(h, rank, world)
        hs = D.HaloStrip(r1 - r0, (w,), kern.max_radius, torch.float32, torch.device("cpu"))
        hs.interior.copy_(torch.from_numpy(img[r0:r1]))
        hs.exchange()
        top, bottom = hs.top, hs.bottom
        ok_rows = np.array_equal(hs.ext.numpy(), img[r0 - top:r1 + bottom])
        full = O.separable_filter_2d(img, kern.radii, kern.weights, threads=2).astype(np.float32)
        errs = []
        for overlap in (False, True):
            got = D.filter_strip(hs, kern, value_bound=255.0, overlap=overlap, _window=_oracle_window)
            errs.append(float(np.abs(got.numpy() - full[r0:r1]).max()))
        slowest = D.max_over_ranks(float(rank + 1))
        q.put((rank, ok_rows, top, bottom, errs, slowest))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,h", [(2, 96), (3, 131), (2, 400)])
def test_row_strip_partition_matches_full_image(world, h):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, 70, 6.0, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    pmax = table_kernel(4, 6.0).max_radius
    for rank, ok_rows, top, bottom, errs, slowest in res:
        assert ok_rows, rank
        assert top == (pmax if rank > 0 else 0)
        assert bottom == (pmax if rank < world - 1 else 0)
        assert max(errs) <= 1e-4, (rank, errs)  # float32 rounding of the float64 band filter
        assert slowest == float(world)


def _thin_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kern = table_kernel(4, 6.0)  # pmax 13
        rows = 40 if rank == 0 else 12  # rank 1's strip is thinner than the halo
        try:
            D.filter_strip(torch.zeros((rows, 50)), kern, value_bound=1.0, _window=_oracle_window)
            q.put((rank, "no error"))
        except ValueError as exc:
            q.put((rank, str(exc)))
    finally:
        dist.destroy_process_group()


def test_thin_strip_raises_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_thin_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all("thinner than the halo" in msg for _, msg in res), res


def test_shard_range_covers_batch():
    for world in (1, 2, 3, 8):
        spans = [D.shard_range(256, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 256
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1
    with pytest.raises(ValueError):
        D.shard_range(10, 2, 2)

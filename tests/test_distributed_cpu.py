"""World-size 2/3 CPU (gloo) tests of the multi-GPU plumbing.

The row-strip partition (config 5) must reproduce the full-image result: each
rank receives its neighbours' halo rows over point-to-point sends, and the
strip filter (here the float64 oracle's band filter, which has the row-window
semantics of sb_separable_filter_2d_window) must equal the same rows of the
whole-image reference.  Batch sharding (config 3) must cover every image once.
The GPU kernels are exercised by tests/test_gpu_parity.py.
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
        local = torch.from_numpy(img[r0:r1].copy())
        ext, top, bottom = D.exchange_halo(local, kern.max_radius)
        ok_rows = np.array_equal(ext.numpy(), img[r0 - top:r1 + bottom])
        got = O.filter_band(ext.numpy(), kern.radii, kern.weights, top, top + (r1 - r0), threads=2)
        full = O.separable_filter_2d(img, kern.radii, kern.weights, threads=2)
        err = float(np.abs(got - full[r0:r1]).max())
        slowest = D.max_over_ranks(float(rank + 1))
        q.put((rank, ok_rows, top, bottom, err, slowest))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,h", [(2, 96), (3, 131)])
def test_row_strip_partition_matches_full_image(world, h):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, 70, 6.0, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    pmax = table_kernel(4, 6.0).max_radius
    for rank, ok_rows, top, bottom, err, slowest in res:
        assert ok_rows, rank
        assert top == (pmax if rank > 0 else 0)
        assert bottom == (pmax if rank < world - 1 else 0)
        assert err <= 1e-9, (rank, err)
        assert slowest == float(world)


def test_shard_range_covers_batch():
    for world in (1, 2, 3, 8):
        spans = [D.shard_range(256, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 256
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1
    with pytest.raises(ValueError):
        D.shard_range(10, 2, 2)

"""Multi-GPU partitions of the filter (one process per GPU, torch.distributed).

Two decompositions, as BASELINE.json's configs ask; the
reference itself only has a 4-thread row-block pool (filtering.py:91-101):

* **batch sharding** (config 3): images are independent, so every rank filters
  its own ``shard_range`` of the batch; there is no data-path collective.
* **row-strip partition** (config 5): one giant image split into horizontal
  strips.  The column pass of a strip's edge rows needs ``pmax`` rows of each
  neighbour (pmax = the largest slice radius); they are exchanged point-to-point
  (``batch_isend_irecv``: NCCL P2P over NVLink on GPUs, gloo on CPU) straight
  into the halo rows of a persistent ``[halo | strip | halo]`` buffer
  (``HaloStrip``), so only the 2 x pmax halo rows move, never the strip.  The
  row-window entry point of the C ABI (``sb_separable_filter_2d_window``) filters
  the strip treating only the global top and bottom as image edges.  With
  ``overlap`` the interior rows (whose column windows stay inside the strip) are
  filtered while the halo rows are in flight, then the two edge bands.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .approx import SliceKernel


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [begin, end) share of ``total`` units for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    return total * rank // world, total * (rank + 1) // world


def _peer(group, rank):
    return dist.get_global_rank(group, rank) if group is not None else rank


class HaloStrip:
    """A rank's strip inside a persistent ``[halo | strip | halo]`` buffer.

    ``interior`` is the strip (rows on dim 0), a view of ``ext``; fill it (or
    build the strip in it) once, then ``exchange`` / ``filter_strip`` move only
    the halo rows.  Rank 0 has no top halo and the last rank no bottom halo (the
    global edges keep the replicate boundary).
    """

    def __init__(self, rows: int, tail_shape: tuple, halo: int, dtype, device, group=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        self.rows = rows
        self.halo = halo
        self.top = halo if self.rank > 0 else 0
        self.bottom = halo if self.rank < self.world - 1 else 0
        self.ext = torch.empty((self.top + rows + self.bottom,) + tuple(tail_shape), dtype=dtype, device=device)
        self.interior = self.ext[self.top:self.top + rows]

    @classmethod
    def wrap(cls, local: torch.Tensor, halo: int, group=None) -> "HaloStrip":
        hs = cls(local.shape[0], tuple(local.shape[1:]), halo, local.dtype, local.device, group)
        hs.interior.copy_(local)
        return hs

    def post_exchange(self):
        """Post the halo sends/receives (returns the requests; ``wait`` them)."""
        h, halo = self.rows, self.halo
        ops = []
        if self.top:
            peer = _peer(self.group, self.rank - 1)
            ops.append(dist.P2POp(dist.isend, self.interior[:halo], peer, self.group))
            ops.append(dist.P2POp(dist.irecv, self.ext[:self.top], peer, self.group))
        if self.bottom:
            peer = _peer(self.group, self.rank + 1)
            ops.append(dist.P2POp(dist.isend, self.interior[h - halo:], peer, self.group))
            ops.append(dist.P2POp(dist.irecv, self.ext[self.top + h:], peer, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def exchange(self):
        for req in self.post_exchange():
            req.wait()


def check_strips(rows: int, halo: int, group=None) -> None:
    """Every strip must be at least ``halo`` rows tall.  Decided collectively (MIN
    over ranks) before any point-to-point op, so either every rank raises or none."""
    world = dist.get_world_size(group)
    if world == 1:
        return
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([rows], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    thinnest = int(t.item())
    if halo > thinnest:
        raise ValueError(f"a strip of {thinnest} rows is thinner than the halo of {halo} rows; use fewer ranks")


def filter_strip(local, kernel: SliceKernel, *, channels_last: bool = False, value_bound=None, group=None,
                 out=None, check: bool = True, overlap=None, _window=None) -> torch.Tensor:
    """Filter this rank's strip of a row-partitioned image (config 5).

    ``local`` is the rank's (rows, W[, C]) CUDA tensor, or a ``HaloStrip`` whose
    interior holds it (no copy of the strip then).  The result equals the same
    rows of ``separable_filter_2d`` of the whole image.  ``overlap`` (default:
    when the strip is at least 32 halos tall, where the edge bands' extra sweep
    rows cost less than the exchange they hide) filters the interior rows before
    waiting for the halo rows.  (``_window`` replaces the row-window filter in the
    CPU tests, which run this decomposition with the oracle.)
    """
    if _window is None:
        from .filtering import separable_filter_window as _window

    halo = kernel.max_radius
    if isinstance(local, HaloStrip):
        hs = local
        if hs.halo != halo:
            raise ValueError("HaloStrip was built for another halo")
    else:
        hs = None
    rows = hs.rows if hs is not None else local.shape[0]
    check_strips(rows, halo, group)
    if hs is None:
        hs = HaloStrip.wrap(local, halo, group)
    h, top = hs.rows, hs.top
    if value_bound is None and hs.ext.dtype in (torch.float32, torch.float64):
        # one bound (hence one quantum) for every rank: the strips then agree bit for bit
        # with the single-image filter
        m = hs.interior.abs().max().to(torch.float64).reshape(1)
        if hs.world > 1:
            if dist.get_backend(group) != "nccl":
                m = m.cpu()
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
        value_bound = float(m.item())
    shape = (h,) + tuple(hs.ext.shape[1:])
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=hs.ext.device)
    if overlap is None:
        overlap = h >= 32 * max(1, halo)
    kw = dict(channels_last=channels_last, value_bound=value_bound, check=check)
    steps = strip_plan(h, top, hs.bottom, halo, overlap and hs.world > 1)
    # the halo rows travel (NCCL's stream) while the steps that do not need them run
    reqs = hs.post_exchange()
    waited = False
    for src0, src1, r0, r1, o0, o1, needs_halo in steps:
        if needs_halo and not waited:
            for req in reqs:
                req.wait()
            waited = True
        _window(hs.ext[src0:src1], kernel, r0, r1, out=out[o0:o1], **kw)
    if not waited:
        for req in reqs:
            req.wait()
    return out


def strip_plan(h: int, top: int, bottom: int, halo: int, overlap: bool):
    """The row-window launches that filter a strip of ``h`` rows stored at rows
    [top, top + h) of its [top halo | strip | bottom halo] buffer.

    Returns ``(src_begin, src_end, row_begin, row_end, out_begin, out_end,
    needs_halo)`` tuples: filter buffer rows [src_begin, src_end) as an image,
    output its rows [row_begin, row_end) into strip rows [out_begin, out_end).
    Without overlap: one launch on the whole buffer after the exchange.  With
    overlap: the interior rows [halo, h - halo) from the strip alone (their column
    windows never leave it), then the two edge bands from the strip plus halo.
    """
    n = top + h + bottom
    if not overlap or h <= 2 * halo:
        return [(0, n, top, top + h, 0, h, True)]
    e0 = top + h - 2 * halo
    return [
        (top, top + h, halo, h - halo, halo, h - halo, False),
        (0, top + 2 * halo, top, top + halo, 0, halo, True),
        (e0, n, halo, 2 * halo, h - halo, h, True),
    ]


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (the bench's timing rule: slowest rank wins)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())

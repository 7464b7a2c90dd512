"""Multi-GPU partitions of the filter (one process per GPU, torch.distributed).

Two decompositions, as BASELINE.json's configs ask:

* **batch sharding** (config 3): images are independent, so every rank filters
  its own images; there is no data-path collective (``shard_range``).
* **row-strip partition** (config 5): one giant image split into horizontal
  strips.  The column pass of a strip's edge rows needs ``pmax`` rows of each
  neighbour (pmax = the largest slice radius); they are exchanged point-to-point
  (``exchange_halo``: ``batch_isend_irecv``, NCCL over NVLink on GPUs, gloo on
  CPU) and the strip is filtered with the row-window variant of the C ABI
  (``sb_separable_filter_2d_window``), which treats only the global top and
  bottom as image edges.  The row pass needs no exchange: strips hold whole
  rows.
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


def exchange_halo(local: torch.Tensor, halo: int, group=None) -> tuple[torch.Tensor, int, int]:
    """Return ``(extended, top, bottom)``: ``local`` (rows on dim 0) with up to
    ``halo`` rows of the previous rank stacked above and of the next rank below.

    Rank 0 gets no top halo and the last rank no bottom halo (global edges keep
    the replicate boundary).  Every strip must have at least ``halo`` rows.
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    h = local.shape[0]
    if halo > h and world > 1:
        raise ValueError(f"strip of {h} rows is thinner than the halo of {halo} rows; use fewer ranks")
    top = halo if rank > 0 else 0
    bottom = halo if rank < world - 1 else 0
    ext = torch.empty((top + h + bottom,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    ext[top:top + h].copy_(local)
    ops = []
    if top:
        peer = dist.get_global_rank(group, rank - 1) if group is not None else rank - 1
        ops.append(dist.P2POp(dist.isend, local[:halo].contiguous(), peer, group))
        ops.append(dist.P2POp(dist.irecv, ext[:top], peer, group))
    if bottom:
        peer = dist.get_global_rank(group, rank + 1) if group is not None else rank + 1
        ops.append(dist.P2POp(dist.isend, local[h - halo:].contiguous(), peer, group))
        ops.append(dist.P2POp(dist.irecv, ext[top + h:], peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return ext, top, bottom


def filter_strip(local: torch.Tensor, kernel: SliceKernel, *, channels_last: bool = False, value_bound=None,
                 group=None, out=None) -> torch.Tensor:
    """Filter this rank's strip of a row-partitioned image (config 5).

    ``local`` is the rank's (rows, W[, C]) CUDA tensor; the result equals the
    same rows of ``separable_filter_2d`` of the whole image.
    """
    from .filtering import separable_filter_window

    ext, top, _ = exchange_halo(local, kernel.max_radius, group)
    return separable_filter_window(ext, kernel, top, top + local.shape[0], channels_last=channels_last,
                                   value_bound=value_bound, out=out, check=False)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (the bench's timing rule: slowest rank wins)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())

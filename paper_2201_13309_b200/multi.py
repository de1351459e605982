"""Multi-GPU plumbing for row-sharded reconstruction.

One process per GPU (torchrun), NCCL through torch.distributed.  The detector rows
are split into contiguous bands; every rank reconstructs its own band with its own
plan (daxm_create with row_begin/row_end) -- there is no data-path collective.
Optional exchanges, timed separately by bench.py:

* ``gather_rows``: all-gather of the output planes [M][rows_g][C] into the full
  [M][R][C] image set (the paper's image_set.depth_resolved);
* ``allreduce_profile``: all-reduce of the M-length depth profile
  (image_set.depth_intensity).

Bands are aligned to the deposit tile height (128 rows) when the split allows it,
so that each band's output is bit-identical to the same rows of a single-GPU run.
This module holds host logic only; with a CPU tensor and the gloo backend it runs
without a GPU (tests/test_multi_gloo.py).
"""
from __future__ import annotations

TILE_ROWS = 128


def row_bands(world: int, n_rows: int, align: int = TILE_ROWS) -> list[tuple[int, int]]:
    """Contiguous [begin, end) row bands, one per rank, covering [0, n_rows).

    Boundaries are multiples of `align` when every band can still get at least one
    aligned block; otherwise an even split (the first tile of a band that starts
    inside a tile then runs the general kernel -- still exact to tolerance).
    """
    if world < 1 or n_rows < world:
        raise ValueError(f"cannot split {n_rows} rows over {world} ranks")
    blocks = n_rows // align
    if align > 1 and blocks >= world:
        cuts = [round(g * blocks / world) * align for g in range(world)] + [n_rows]
    else:
        cuts = [g * n_rows // world for g in range(world)] + [n_rows]
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def my_band(rank: int, world: int, n_rows: int, align: int = TILE_ROWS) -> tuple[int, int]:
    return row_bands(world, n_rows, align)[rank]


def gather_rows(out_band, bands, group=None):
    """All-gather [M][rows_g][C] bands (unequal heights allowed) into [M][R][C] on every rank."""
    import torch
    import torch.distributed as dist
    world = len(bands)
    M, _, C = out_band.shape
    hmax = max(e - b for b, e in bands)
    pad = torch.zeros((M, hmax, C), dtype=out_band.dtype, device=out_band.device)
    pad[:, : out_band.shape[1]] = out_band
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, M, hmax, C), dtype=out_band.dtype, device=out_band.device)
        dist.all_gather_into_tensor(buf, pad.contiguous(), group=group)
    else:  # gloo: no all_gather_into_tensor; exchange through host memory
        pad = pad.cpu()
        buf = torch.empty((world, M, hmax, C), dtype=out_band.dtype)
        dist.all_gather(list(buf.unbind(0)), pad.contiguous(), group=group)
        buf = buf.to(out_band.device)
    full = torch.empty((M, bands[-1][1], C), dtype=out_band.dtype, device=out_band.device)
    for g, (b, e) in enumerate(bands):
        full[:, b:e] = buf[g, :, : e - b]
    return full


def hist_allreduce(group=None, device=None):
    """The daxm_select_cutoff_sharded callback for torch.distributed: sums a uint64 numpy
    histogram over the ranks in place (through `device` for NCCL, in host memory for gloo).
    Counts stay below 2**63, so the int64 all-reduce is exact."""
    import numpy as np
    import torch
    import torch.distributed as dist

    def reduce(hist):
        t = torch.from_numpy(hist.view(np.int64).copy())
        if dist.get_backend(group) == "nccl":
            t = t.to(device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        hist.view(np.int64)[:] = t.cpu().numpy()
    return reduce


def select_cutoff(plan, stack_band, fraction, n_rows, n_cols, group=None, stream=None):
    """Pixel percentage (reading R14) over the whole detector when each rank holds
    one row band: the global k-th largest I_0, identical on every rank (one 256-bin histogram
    all-reduce per radix digit).  With one rank this is plan.select_cutoff."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return plan.select_cutoff(stack_band, fraction, stream)
    return plan.select_cutoff_sharded(stack_band, fraction, n_rows * n_cols,
                                      hist_allreduce(group, stack_band.device), stream)


def allreduce_profile(profile, group=None):
    """Sum the per-rank depth profiles (M,) in place and return it."""
    import torch.distributed as dist
    dist.all_reduce(profile, op=dist.ReduceOp.SUM, group=group)
    return profile


def max_over_ranks(values, device=None, group=None):
    """Element-wise max of a list of floats over ranks (the bench's timing rule)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if dist.get_backend(group) != "nccl":
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()

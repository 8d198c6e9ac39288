"""Multi-GPU plumbing: z-slab sharding of the build, replicated-field queries.

The build partitions voxels: every voxel's factor is independent
(field.py:617-642 writes disjoint rows), so each rank builds a contiguous range
of the INTERNAL z-major voxel index — a z-slab, split by voxel count rather
than whole planes — after one NCCL broadcast of the landmarks.  There is no
collective in the inner loop.  An optional all-gather replicates the field for
queries; queries are sharded by contiguous pose ranges against the replica.
Per-voxel landmark order is fixed, so the sharded build is bit-identical to the
single-GPU build.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def slab_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of `total` units for `rank` (sizes differ by <= 1)."""
    base, rem = divmod(int(total), int(world))
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def broadcast_points(points, device, src: int = 0) -> torch.Tensor:
    """One broadcast of the (N,3) float64 landmarks from `src` to every rank."""
    if dist.get_rank() == src:
        t = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64)).to(device)
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
    else:
        n = torch.zeros(1, dtype=torch.int64, device=device)
    dist.broadcast(n, src=src)
    if dist.get_rank() != src:
        t = torch.empty((int(n.item()), 3), dtype=torch.float64, device=device)
    dist.broadcast(t, src=src)
    return t


def gather_slabs(local_rows: torch.Tensor, total_rows: int) -> torch.Tensor:
    """All-gather the ranks' slab rows into the full (total_rows, width) field on every rank."""
    world = dist.get_world_size()
    width = local_rows.shape[1]
    sizes = [slab_range(total_rows, world, r) for r in range(world)]
    maxr = max(e - b for b, e in sizes)
    pad = torch.zeros((maxr, width), dtype=local_rows.dtype, device=local_rows.device)
    pad[: local_rows.shape[0]] = local_rows
    buf = torch.empty((world * maxr, width), dtype=local_rows.dtype, device=local_rows.device)
    dist.all_gather_into_tensor(buf, pad)
    parts = [buf[r * maxr: r * maxr + (e - b)] for r, (b, e) in enumerate(sizes)]
    return torch.cat(parts, dim=0)


def build_sharded(points, config, model, factor_kind: str, sigma: float = 1.0, device=None, replicate: bool = False,
                  row_builder=None):
    """z-slab build on this rank.  Returns (v_begin, v_end, rows64, rows32, full64_or_None).

    `row_builder(points_dev, v_begin, v_end) -> (rows64, rows32)` defaults to the CUDA build;
    tests substitute the CPU oracle to check the partition/gather logic under gloo.
    """
    from .field import _grid_of, build_rows
    from .visibility import model_from_reference

    config = _grid_of(config)
    model = model_from_reference(model)
    rank, world = dist.get_rank(), dist.get_world_size()
    pts = broadcast_points(points if rank == 0 else None, device)
    v0, v1 = slab_range(config.voxel_count, world, rank)
    if row_builder is None:
        rows64, rows32 = build_rows(pts, model, factor_kind == "trace", sigma, device, grid=config, v_begin=v0,
                                    v_end=v1)
    else:
        rows64, rows32 = row_builder(pts, v0, v1)
    full = gather_slabs(rows64, config.voxel_count) if replicate else None
    return v0, v1, rows64, rows32, full

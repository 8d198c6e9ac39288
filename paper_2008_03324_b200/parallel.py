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
        if isinstance(points, torch.Tensor):  # e.g. pinned host memory: one direct H2D copy
            t = points.to(device=device, dtype=torch.float64).reshape(-1, 3).contiguous()
        else:
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


def build_field(points, config, model, factor_kind: str = "info", sigma: float = 1.0, device=None,
                replicate: bool = True):
    """Sharded build through the public Field type (Field.build(..., process_group=...)):
    rank 0's landmarks broadcast once, each rank builds its z-slab (no collective in the
    inner loop), then either an all-gather of the FP64 rows gives every rank the whole dense
    field (replicate=True), or the rank keeps its slab as a Field over the global grid
    (voxels of other ranks read as absent)."""
    from .field import Field, GpVisibility, _grid_of

    config = _grid_of(config)
    v0, v1, rows64, rows32, full = build_sharded(points, config, model, factor_kind, sigma, device, replicate)
    from .visibility import model_from_reference

    model = model_from_reference(model)
    if replicate:
        f32 = full.float() if isinstance(model, GpVisibility) else None
        return Field(config, model, factor_kind, sigma, full, f32, None, dense=True)
    occ3 = config.index3_of_internal(np.arange(v0, v1)).astype(np.int32)
    return Field(config, model, factor_kind, sigma, rows64, rows32, occ3, dense=False)


# ── slab-routed queries (fields larger than one GPU's HBM) ─────────────────
# each rank keeps the z-planes it owns plus a one-plane halo (the upper
# trilinear corner), queries are routed to the owner of their base z-index with an
# all-to-all of (pose, id) and the results come back the same way.  The owner queries
# its slab through a slots map over the GLOBAL grid, so corner lookup, weights and
# status use the full grid's geometry and every result is bit-identical to a query on
# the unsharded field.

QUERY_WIDTHS = {"trace": 1, "trace_grad": 6, "fim": 36, "fim_grad": 216, "det": 1, "det_grad": 6, "lmin": 1,
                "lmin_grad": 6, "status": 1}


def plane_range(nz: int, world: int, rank: int) -> tuple[int, int]:
    """z-planes [z0, z1) owned by `rank` (plane-aligned split for routed queries)."""
    return slab_range(nz, world, rank)


def slab_rows_range(config, world: int, rank: int) -> tuple[int, int, int, int]:
    """(z0, z1, v_begin, v_end): owned planes and the internal z-major row range of the
    owned planes plus the one-plane halo above them."""
    nx, ny, nz = (int(d) for d in config.dims)
    z0, z1 = plane_range(nz, world, rank)
    zh = min(z1 + 1, nz)
    return z0, z1, z0 * nx * ny, zh * nx * ny


def query_owners(positions, config, world: int, trilinear: bool):
    """Owner rank of each query: the rank whose planes hold its base z-index (trilinear:
    floor((z - o_z)/vs - 0.5), so both corner planes are on the owner; nearest:
    floor((z - o_z)/vs)); out-of-field queries go to the nearest plane's owner, which
    reports the out-of-field status.  numpy in -> numpy out; torch in -> torch out on the
    same device.  The FP64 expression is the query kernels' locate (kernels.py:628-635,
    679-702) operation for operation, so the owner always holds the corners it reads."""
    nz = int(config.dims[2])
    starts = [plane_range(nz, world, r)[0] for r in range(world)]
    hi = max(nz - (2 if trilinear else 1), 0)
    if isinstance(positions, torch.Tensor):
        g = (positions[:, 2].to(torch.float64) - float(config.origin[2])) / float(config.voxel_size)
        if trilinear:
            g = g - 0.5
        bz = torch.clamp(torch.floor(g), 0, hi).to(torch.int64)
        st = torch.tensor(starts, dtype=torch.int64, device=positions.device)
        return torch.searchsorted(st, bz, right=True) - 1
    g = (np.asarray(positions, dtype=np.float64)[:, 2] - config.origin[2]) / config.voxel_size
    if trilinear:
        g = g - 0.5
    bz = np.clip(np.floor(g), 0, hi).astype(np.int64)
    return np.searchsorted(np.array(starts), bz, side="right") - 1


def route_queries(positions, axes, config, trilinear: bool, query_fn, outputs, device=None) -> dict:
    """Run this rank's queries on their owners.  `query_fn(pos (n,3), axes (n,3)) ->
    {name: (n, width) tensor or array}` answers queries against this rank's slab; `outputs`
    names the entries of QUERY_WIDTHS wanted.  Returns {name: (Q, width) float64 tensor} in
    the caller's order, on `device` (default: the device of `positions` if it is a tensor,
    else the CPU).  Every exchanged buffer (counts, requests, results) is a tensor on that
    device, so the collectives run on NCCL for CUDA tensors and on gloo for CPU tensors;
    the only host transfer is the split sizes all_to_all_single needs.  Collectives: one
    all_to_all_single of the counts, one of the requests, one of the results."""
    world = dist.get_world_size()
    if device is None:
        device = positions.device if isinstance(positions, torch.Tensor) else torch.device("cpu")
    pos = torch.as_tensor(positions, dtype=torch.float64).to(device).reshape(-1, 3)
    ax = torch.as_tensor(axes, dtype=torch.float64).to(device).reshape(-1, 3)
    owner = query_owners(pos, config, world, trilinear)
    order = torch.argsort(owner, stable=True)
    send_counts = torch.bincount(owner, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    sc, rc = send_counts.tolist(), recv_counts.tolist()
    req = torch.cat([pos[order], ax[order]], dim=1).contiguous()
    got = torch.empty((sum(rc), 6), dtype=torch.float64, device=device)
    dist.all_to_all_single(got, req, output_split_sizes=rc, input_split_sizes=sc)
    names = [n for n in QUERY_WIDTHS if n in outputs or n == "status"]
    width = sum(QUERY_WIDTHS[n] for n in names)
    n_got = got.shape[0]
    if n_got:
        res = query_fn(got[:, :3].contiguous(), got[:, 3:].contiguous())
        packed = torch.cat([torch.as_tensor(res[n]).to(device=device, dtype=torch.float64).reshape(n_got, -1)
                            for n in names], dim=1).contiguous()
    else:
        packed = torch.zeros((0, width), dtype=torch.float64, device=device)
    back = torch.empty((pos.shape[0], width), dtype=torch.float64, device=device)
    dist.all_to_all_single(back, packed, output_split_sizes=sc, input_split_sizes=rc)
    out = torch.empty_like(back)
    out[order] = back
    result, col = {}, 0
    for n in names:
        result[n] = out[:, col:col + QUERY_WIDTHS[n]]
        col += QUERY_WIDTHS[n]
    return result


def build_slab_field(points, config, model, factor_kind: str, sigma: float = 1.0, device=None):
    """This rank's slab of a z-sharded field (owned planes + one-plane halo) as a device
    Field whose slots map the GLOBAL grid (voxels of other ranks read as absent)."""
    from .field import Field, _grid_of, build_rows
    from .visibility import model_from_reference

    config = _grid_of(config)
    model = model_from_reference(model)
    rank, world = dist.get_rank(), dist.get_world_size()
    pts = broadcast_points(points if rank == 0 else None, device)
    _, _, v0, v1 = slab_rows_range(config, world, rank)
    rows64, rows32 = build_rows(pts, model, factor_kind == "trace", sigma, device, grid=config, v_begin=v0, v_end=v1)
    occ3 = config.index3_of_internal(np.arange(v0, v1)).astype(np.int32)
    return Field(config, model, factor_kind, sigma, rows64, rows32, occ3, dense=False)


def query_slab_field(slab_field, positions, axes, mode: str = "trilinear", outputs=("trace", "full"),
                     grad: bool = False) -> dict:
    """Slab-routed query (see route_queries) answered on each owner's device Field."""
    outs = set(outputs)
    names = {"trace"} if "trace" in outs else set()
    if "full" in outs:
        names.add("fim")
    names |= outs & {"det", "lmin"}
    if grad:
        names |= {n + "_grad" for n in list(names)}
    dev = slab_field.device

    def fn(p, a):  # device tensors in, device tensors out
        r = slab_field.query_device(p, a, mode, trace="trace" in outs, full="full" in outs, det="det" in outs,
                                    lmin="lmin" in outs, grad=grad)
        return {k: v.reshape(v.shape[0], -1) for k, v in r.items()}

    return route_queries(positions, axes, slab_field.config, mode == "trilinear", fn, names, device=dev)

"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): landmark broadcast, z-slab
partition, all-gather replication.  The per-rank compute is the CPU oracle standing in
for the CUDA build (test seam `row_builder`), so the assembled field must equal the
single-process oracle field bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_03324_b200.parallel import slab_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        import paper_2008_03324_b200 as F
        from paper_2008_03324_b200.parallel import build_sharded

        rng = np.random.default_rng(0)
        pts = rng.uniform([-2, -2, 0], [2, 2, 2], size=(120, 3)) if rank == 0 else None
        grid = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([5, 4, 3]))
        model = F.build_quad_model()
        # internal z-major centres, so slab rows line up with the device layout
        cz = grid.center_of(grid.index3_of_internal(np.arange(grid.voxel_count)))

        def row_builder(p, v0, v1):
            rows = O.build_quad_factors(cz[v0:v1], p.numpy(), 1.0, model.k2, model.k1, model.k0, True)
            return torch.from_numpy(rows), None

        v0, v1, rows, _, full = build_sharded(pts, grid, model, "trace", device=torch.device("cpu"),
                                              replicate=True, row_builder=row_builder)
        if rank == 0:
            ref = O.build_quad_factors(cz, rng_pts(), 1.0, model.k2, model.k1, model.k0, True)
            np.save(result_path, np.stack([full.numpy(), ref]))
    finally:
        dist.destroy_process_group()


def rng_pts():
    return np.random.default_rng(0).uniform([-2, -2, 0], [2, 2, 2], size=(120, 3))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_build_matches_single_process(tmp_path, world):
    out = str(tmp_path / "res.npy")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    full, ref = np.load(out)
    assert np.array_equal(full, ref)


def test_slab_range_partition():
    for total in (0, 1, 7, 137781, 25351101):
        for world in (1, 2, 3, 4, 8):
            r = [slab_range(total, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == total
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            sizes = [e - b for b, e in r]
            assert max(sizes) - min(sizes) <= 1


def _routed_worker(rank, world, port, result_path, trilinear):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        import paper_2008_03324_b200 as F
        from paper_2008_03324_b200.parallel import query_owners, route_queries, slab_rows_range

        grid = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([4, 3, 7]))
        model = F.build_quad_model()
        om = ("quad", model.k2, model.k1, model.k0)
        pts = rng_pts()
        centers = grid.centers()  # reference x-major order
        full = O.build_quad_factors(centers, pts, 1.0, model.k2, model.k1, model.k0, False)
        # this rank's slab: owned planes + halo, in the reference layout, with slots over
        # the global grid (other ranks' voxels absent) — what the device Field holds
        _, _, v0, v1 = slab_rows_range(grid, world, rank)
        idx3 = grid.index3_of_internal(np.arange(v0, v1))
        lin = grid.linear_index(idx3)
        slots = np.full(grid.voxel_count, -1, np.int32)
        slots[lin] = np.arange(v1 - v0, dtype=np.int32)
        slab = full[lin]

        def query_fn(p, a):  # CPU tensors in (gloo), numpy arrays out
            p, a = p.numpy(), a.numpy()
            fim, st = O.query_fim_batch(slots, slab, grid.origin, grid.voxel_size, grid.dims, p, a, om, trilinear)
            tr, _ = O.metric_batch(slots, slab, grid.origin, grid.voxel_size, grid.dims, p, a, om, "trace", False,
                                   trilinear)
            return {"fim": fim.reshape(-1, 36), "trace": tr[:, None], "status": st[:, None].astype(np.float64)}

        rng = np.random.default_rng(100 + rank)
        c = grid.centers()
        pos = rng.uniform(c[0] - 0.4, c[-1] + 0.4, size=(50 + 7 * rank, 3))
        ax = rng.standard_normal((pos.shape[0], 3))
        ax /= np.linalg.norm(ax, axis=1, keepdims=True)
        got = {k: v.numpy() for k, v in route_queries(pos, ax, grid, trilinear, query_fn, {"trace", "fim"}).items()}
        own_np = query_owners(pos, grid, world, trilinear)
        own_t = query_owners(torch.from_numpy(pos), grid, world, trilinear).numpy()
        assert np.array_equal(own_np, own_t)  # torch routing == numpy routing, bit for bit
        all_slots = np.arange(grid.voxel_count, dtype=np.int32)
        fim, st = O.query_fim_batch(all_slots, full, grid.origin, grid.voxel_size, grid.dims, pos, ax, om, trilinear)
        tr, _ = O.metric_batch(all_slots, full, grid.origin, grid.voxel_size, grid.dims, pos, ax, om, "trace", False,
                               trilinear)
        ok = (np.array_equal(got["fim"], fim.reshape(-1, 36)) and np.array_equal(got["trace"][:, 0], tr)
              and np.array_equal(got["status"][:, 0], st.astype(np.float64)))
        np.save(result_path + f".{rank}.npy", np.array([ok, (st == 0).sum()]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("trilinear", [True, False])
def test_slab_routed_queries_match_full_field(tmp_path, world, trilinear):
    """SURVEY 8(e) slab-routed queries: per-rank z-slabs (+1 halo plane), all-to-all of
    requests and results; bit-identical to querying the unsharded field."""
    out = str(tmp_path / "routed")
    mp.start_processes(_routed_worker, args=(world, _free_port(), out, trilinear), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        ok, n_in = np.load(out + f".{r}.npy")
        assert ok and n_in > 0

"""Configs 4 and 5 of SURVEY §8(d) on one B200.

Config 4: 1 000 000 clustered float32 landmarks (scenes.config4, seed 3).
  * GP-70 full-6x6 build of a z-slab of the 251x251x51 @0.4 m grid and GP-70 trace
    build of a z-slab of the 501x501x101 @0.2 m grid (internal z-major rows, the unit a
    GPU shard builds); pairs/s and the extrapolated whole-config time on 1 and 8 GPUs;
    parity of sampled voxels against the C oracle (test infrastructure).
Config 5 (--full): the whole config-4 GP-70 info field (3.2e12 pairs, ~57 GB of HBM),
  then B-spline query batches (64 poses each, scenes.bspline_trajectory_batch, seed 4):
  full 6x6 + trace + analytic gradient, queries/s; parity of a query sample against the
  oracle on a cropped field.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC
from oracle import oracle as O

ap = argparse.ArgumentParser()
ap.add_argument("--info-planes", type=int, default=2)
ap.add_argument("--trace-planes", type=int, default=1)
ap.add_argument("--n-points", type=int, default=1000000)
ap.add_argument("--full", action="store_true", help="build the whole config-4 info field and run config 5")
ap.add_argument("--nq", type=int, default=100_000_000)
ap.add_argument("--parity-voxels", type=int, default=16)
a = ap.parse_args()
dev = torch.device("cuda")
gp70 = F.build_gp_model(70)
pts_np = SC.cluster_mixture(a.n_points)
pts = torch.tensor(pts_np, device=dev)
N = pts_np.shape[0]
rng = np.random.default_rng(0)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3


def slab_probe(kind, planes):
    w = SC.config4(kind, 1)
    grid = F.GridConfig(*w.grid)
    nx, ny, nz = (int(d) for d in grid.dims)
    z0 = nz // 2
    v0, v1 = z0 * nx * ny, (z0 + planes) * nx * ny
    dm = FD._DeviceModel(gp70, dev)
    trace = kind == "trace"
    FD.build_rows(pts, gp70, trace, 1.0, dev, grid=grid, v_begin=v0, v_end=v0 + nx, dmodel=dm)  # warm-up
    (s64, _), t = timed(lambda: FD.build_rows(pts, gp70, trace, 1.0, dev, grid=grid, v_begin=v0, v_end=v1,
                                              dmodel=dm, f32_copy=False))
    pairs = (v1 - v0) * N
    rate = pairs / t
    total = grid.voxel_count * N
    print(f"config4 GP-70 {kind}: {v1 - v0} voxels x {N} landmarks in {t:.2f} s = {rate:.3e} pairs/s; "
          f"whole config ({total:.3e} pairs) extrapolated {total / rate:.0f} s on 1 GPU, "
          f"{total / rate / 8:.0f} s on 8", flush=True)
    # parity on sampled rows (internal z-major -> centres)
    sel = np.sort(rng.choice(v1 - v0, a.parity_voxels, replace=False))
    idx3 = grid.index3_of_internal(v0 + sel)
    cen = grid.center_of(idx3)
    t0 = time.time()
    ref = O.build_gp_factors(cen, pts_np, 1.0, gp70.samples, gp70.kinv, gp70.k_s, np.cos(gp70.alpha), trace)
    ot = time.time() - t0
    sub = FD.Field(grid, gp70, kind, 1.0, s64[torch.as_tensor(sel, device=dev)].contiguous(), None,
                   idx3.astype(np.int32), dense=False)
    mine = sub.factors
    if trace:
        err = np.linalg.norm(mine - ref, axis=1) / np.linalg.norm(ref, axis=1)
    else:
        err = np.abs(mine - ref).max(axis=1) / np.linalg.norm(ref, axis=1)
    print(f"  parity on {len(sel)} sampled voxels vs oracle: max {err.max():.3e} "
          f"({'per-voxel rel L2' if trace else 'max entry / voxel Frobenius'}; oracle {ot:.1f} s)", flush=True)
    return rate


slab_probe("info", a.info_planes)
slab_probe("trace", a.trace_planes)

if a.full:
    w = SC.config4("info", 1)
    grid = F.GridConfig(*w.grid)
    f, t = timed(lambda: F.Field.build(pts, grid, gp70, "info"))
    print(f"config4 GP-70 info, whole grid: {grid.voxel_count * N:.3e} pairs in {t:.1f} s = "
          f"{grid.voxel_count * N / t:.3e} pairs/s; field {f.memory_stats()['device_bytes'] / 1e9:.1f} GB on device",
          flush=True)
    _, t_tab = timed(lambda: f.trace_table())  # one-time FP64 trace table (first trace query builds it)
    print(f"config5: FP64 trace table of the config-4 field built in {t_tab * 1e3:.1f} ms (once per field)", flush=True)
    qrng = np.random.default_rng(4)
    chunk = 1 << 20
    batches = chunk // 64
    done, busy, nin = 0, 0.0, 0
    out = {}
    first = None
    while done < a.nq:
        pos, rot = SC.bspline_trajectory_batch(qrng, batches)
        p = torch.tensor(pos, device=dev)
        ax = torch.tensor(np.ascontiguousarray(rot[:, :, 2]), device=dev)
        res, t = timed(lambda: f.query_device(p, ax, "trilinear", trace=True, full=True, grad=True, out=out))
        busy += t
        nin += int((res["status"] == 0).sum())
        if first is None:
            first = (pos[:16].copy(), rot[:16].copy(), res["trace"][:16].cpu().numpy(),
                     res["fim"][:16].cpu().numpy().reshape(-1, 6, 6), res["status"][:16].cpu().numpy())
        done += pos.shape[0]
    print(f"config5: {done} B-spline queries (64/batch), full+trace+grad: {busy:.2f} s device time = "
          f"{done / busy:.3e} queries/s, in-field fraction {nin / done:.3f}", flush=True)
    pos, rot, tr, fim, st = first
    need = sorted({int(i) for p_ in pos for i in O.trilinear(grid.origin, grid.voxel_size, grid.dims, p_)[0]})
    if need:
        need = np.array(need)
        t0 = time.time()
        rows = O.build_gp_factors(grid.centers()[need], pts_np, 1.0, gp70.samples, gp70.kinv, gp70.k_s,
                                  np.cos(gp70.alpha), False)
        slots = np.full(grid.voxel_count, -1, np.int32)
        slots[need] = np.arange(len(need), dtype=np.int32)
        ax = np.ascontiguousarray(rot[:, :, 2])
        mt = ("gp", gp70.samples, gp70.params.sigma2, gp70.params.length_scale)
        rt, rst = O.metric_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, pos, ax, mt, "trace", False, True)
        rf, _ = O.query_fim_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, pos, ax, mt, True)
        ok = rst == 0
        et = np.abs(tr[ok] - rt[ok]) / np.abs(rt[ok])
        ef = np.linalg.norm((fim[ok] - rf[ok]).reshape(ok.sum(), -1), axis=1) / np.linalg.norm(
            rf[ok].reshape(ok.sum(), -1), axis=1)
        print(f"  config5 parity on {ok.sum()} in-field queries: status equal {np.array_equal(st, rst)}, trace rel "
              f"max {et.max():.2e}, 6x6 relF max {ef.max():.2e} (oracle {time.time() - t0:.0f} s)", flush=True)

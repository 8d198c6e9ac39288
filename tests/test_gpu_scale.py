"""BASELINE configs 4 and 5 at their full sizes (SURVEY §8(c) "scale workarounds").

Config 4: 1 000 000 clustered float32 landmarks; the trace grid 501x501x101 @0.2 m and the
full-info grid 251x251x51 @0.4 m.  The GPU builds rows for sampled voxels (random + the
grid's extreme corners) through the same kernels as whole-grid builds, compared with the
C oracle (the reference's algorithm) on the same voxels.

Config 5: one 64-pose B-spline batch of the trajectory-optimisation stream against the
config-4 full-info field, restricted to the voxels its queries touch (a cropped field,
exactly as the reference's Field would hold them): statuses bit-exact, trace and 6x6
within 1e-4, and the analytic pose gradients against central differences of the
oracle's FP64 queries on the oracle's own rows.
"""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes
from paper_2008_03324_b200.geometry import so3_exp
from tests._helpers import info_rel_fro, models_from_golden, oracle_field, oracle_model, trace_rel_l2

pytestmark = pytest.mark.gpu
TRACE_TOL, INFO_TOL, Q_TOL = 1e-5, 1e-4, 1e-4


@pytest.fixture(scope="module")
def models(g_models):
    return models_from_golden(g_models)


@pytest.fixture(scope="module")
def points4():
    return scenes.config4("info").points  # the same 1 M landmarks serve both grids


@pytest.mark.parametrize("mname", ["quad", "gp70"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_config4_sampled_voxels(oracle, models, points4, mname, kind):
    w = scenes.config4(kind, n_points=0)
    grid = F.GridConfig(*w.grid)
    rng = np.random.default_rng(12)
    nx, ny, nz = (int(d) for d in grid.dims)
    idx3 = np.vstack([grid.index3_of(rng.choice(grid.voxel_count, 5, replace=False)),
                      [[0, 0, 0], [nx - 1, ny - 1, nz - 1], [nx // 2, ny // 2, nz // 2]]])
    cen = grid.center_of(idx3)
    m = models[mname]
    dev = torch.device("cuda")
    s64, _ = FD.build_rows(torch.tensor(points4, device=dev), m, kind == "trace", 1.0, dev,
                           centers=torch.tensor(cen, device=dev))
    fld = FD.Field(grid, m, kind, 1.0, s64, None, idx3.astype(np.int32), dense=False)
    ref = oracle_field(oracle, m, cen, points4, kind)
    err = trace_rel_l2(fld.factors, ref) if kind == "trace" else info_rel_fro(fld.factors, ref)
    tol = TRACE_TOL if kind == "trace" else INFO_TOL
    if mname == "quad":
        tol = 1e-12  # FP64 per pair
    print(f"config4 {mname} {kind}: max err {err.max():.2e}")
    assert err.max() <= tol, err.max()


def _cropped(oracle, grid, pos):
    need = np.array(sorted({int(i) for p in pos for i in oracle.trilinear(grid.origin, grid.voxel_size, grid.dims, p)[0]
                            if i >= 0}))
    slots = np.full(grid.voxel_count, -1, np.int32)
    slots[need] = np.arange(len(need), dtype=np.int32)
    return need, slots


def test_config5_bspline_batch(oracle, models, points4):
    w = scenes.config4("info", n_points=0)
    grid = F.GridConfig(*w.grid)
    rng = np.random.default_rng(4)
    pos, rot = scenes.bspline_trajectory_batch(rng, 1)  # one 64-pose batch of the config-5 stream
    g = (pos - grid.origin) / grid.voxel_size - 0.5
    frac = g - np.floor(g)
    keep = ((frac > 1e-3) & (frac < 1 - 1e-3)).all(axis=1)  # >= 2h from cell faces (central differences)
    pos, rot = pos[keep][:6], rot[keep][:6]
    q = pos.shape[0]
    assert q >= 4
    need, slots = _cropped(oracle, grid, pos)
    m = models["gp70"]
    dev = torch.device("cuda")
    cen = grid.centers()[need]
    s64, s32 = FD.build_rows(torch.tensor(points4, device=dev), m, False, 1.0, dev, centers=torch.tensor(cen, device=dev))
    fld = FD.Field(grid, m, "info", 1.0, s64, s32, grid.index3_of(need).astype(np.int32), dense=False)
    res = fld.query_batch(pos, rotations=rot, outputs=("trace", "full"), grad=True, to_numpy=True)
    rows = oracle_field(oracle, m, cen, points4, "info")
    om = oracle_model(m)

    def ev(p, r):
        ax = np.ascontiguousarray(r[:, :, 2])
        tr, st = oracle.metric_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, p, ax, om, "trace", False, True)
        fim, _ = oracle.query_fim_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, p, ax, om, True)
        return tr, fim, st

    rt, rf, st = ev(pos, rot)
    assert np.array_equal(res["in_field"], st == 0) and res["in_field"].all()
    assert (np.abs(res["trace"] - rt) / np.abs(rt)).max() <= Q_TOL
    e = np.linalg.norm((res["fim"] - rf).reshape(q, -1), axis=1) / np.linalg.norm(rf.reshape(q, -1), axis=1)
    assert e.max() <= Q_TOL
    # analytic gradients vs central differences (h = 1e-6) of the oracle queries
    h = 1e-6
    g_tr = np.zeros((q, 6))
    g_fim = np.zeros((q, 6, 6, 6))
    for j in range(6):
        if j < 3:
            d = np.zeros(3)
            d[j] = h
            a, b = ev(pos + d, rot), ev(pos - d, rot)
        else:
            wv = np.zeros(3)
            wv[j - 3] = h
            a = ev(pos, np.einsum("ij,qjk->qik", so3_exp(wv), rot))
            b = ev(pos, np.einsum("ij,qjk->qik", so3_exp(-wv), rot))
        g_tr[:, j] = (a[0] - b[0]) / (2 * h)
        g_fim[:, j] = (a[1] - b[1]) / (2 * h)
    et = np.linalg.norm(res["trace_grad"] - g_tr, axis=1) / np.linalg.norm(g_tr, axis=1)
    print(f"config5 sample: trace rel {(np.abs(res['trace'] - rt) / np.abs(rt)).max():.2e}, 6x6 relF {e.max():.2e}, "
          f"trace grad {et.max():.2e}", end="")
    assert et.max() <= Q_TOL, et.max()
    gf = res["fim_grad"].reshape(q, 6, 6, 6)
    ef = np.linalg.norm((gf - g_fim).reshape(q, -1), axis=1) / np.linalg.norm(g_fim.reshape(q, -1), axis=1)
    print(f", 6x6 grad {ef.max():.2e}")
    assert ef.max() <= Q_TOL, ef.max()

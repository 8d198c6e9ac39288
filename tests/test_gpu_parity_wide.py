"""Round-2 parity widening (SURVEY.md §8(c) sampling plan), CUDA path through the C ABI.

* A10 indexing: fif_locate corner indices / weights / status bit-exact against the
  reference's own outputs (golden nearest_index, trilinear_idx_w) and the oracle on the
  config-1 / config-2 grids at edge positions (exact centres, cell faces, last centre,
  one ulp either side of the grid box).
* A14 query_factor against the reference's Field.query_factor (golden).
* Config 1: all 1 000 seed-1 queries (trace + analytic gradient) for GP-70 and quad.
* Config 2: >= 1 000 random + >= 1 000 boundary voxels of the GP-70 / quad info build;
  10 000 queries (query parity on the field's own rows) and 1 000 FD gradients.
* Config 3: 10 000 poses x 20 000 landmarks, masks bit-exact (2e8 pairs).
* Config 4: >= 256 voxels per kind incl. both sides of every 2/4/8-way z-slab seam,
  built in grid (slab) mode exactly as the sharded build runs.
* Config 5: >= 1 000 B-spline query values + 64 FD gradients on the config-4 field.
* A16 planner variant: pc_metric_yaw_batch / ExactInfoRepr vs the reference.

Tolerances (BASELINE north_star): trace PIF per-voxel relative L2 <= 1e-5; full PIF
max-entry <= 1e-4 x voxel Frobenius; query values and gradients <= 1e-4 relative;
indices, statuses and masks bit-exact.
"""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes
from paper_2008_03324_b200.geometry import so3_exp
from paper_2008_03324_b200.parallel import slab_range
from tests._helpers import info_rel_fro, models_from_golden, oracle_field, oracle_model, trace_rel_l2

pytestmark = pytest.mark.gpu
TRACE_TOL, INFO_TOL, Q_TOL = 1e-5, 1e-4, 1e-4
DEV = "cuda"


@pytest.fixture(scope="module")
def models(g_models):
    return models_from_golden(g_models)


def _err(kind, mine, ref):
    return trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)


def _tol(kind):
    return TRACE_TOL if kind == "trace" else INFO_TOL


def _field_on_rows(grid, model, kind, ref_rows, lin):
    """A device Field holding the given reference-layout rows at linear indices `lin`."""
    s64 = torch.tensor(FD._from_reference_rows(ref_rows, model, kind), device=DEV)
    s32 = s64.float() if isinstance(model, F.GpVisibility) else None
    return FD.Field(grid, model, kind, 1.0, s64, s32, grid.index3_of(lin).astype(np.int32), dense=False)


def _oracle_query(oracle, slots, rows, grid, model, kind, pos, rots, full):
    ax = np.ascontiguousarray(rots[:, :, 2])
    tr, st = oracle.metric_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, pos, ax, oracle_model(model),
                                 "trace", kind == "trace", True)
    fim = None
    if full:
        fim, _ = oracle.query_fim_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, pos, ax,
                                        oracle_model(model), True)
    return tr, fim, st


def _fd(oracle, slots, rows, grid, model, kind, pos, rots, full, h=1e-6):
    q = pos.shape[0]
    g_tr = np.zeros((q, 6))
    g_fim = np.zeros((q, 6, 6, 6)) if full else None
    for j in range(6):
        if j < 3:
            d = np.zeros(3)
            d[j] = h
            a = _oracle_query(oracle, slots, rows, grid, model, kind, pos + d, rots, full)
            b = _oracle_query(oracle, slots, rows, grid, model, kind, pos - d, rots, full)
        else:
            w = np.zeros(3)
            w[j - 3] = h
            a = _oracle_query(oracle, slots, rows, grid, model, kind, pos, np.einsum("ij,qjk->qik", so3_exp(w), rots),
                              full)
            b = _oracle_query(oracle, slots, rows, grid, model, kind, pos, np.einsum("ij,qjk->qik", so3_exp(-w), rots),
                              full)
        g_tr[:, j] = (a[0] - b[0]) / (2 * h)
        if full:
            g_fim[:, j] = (a[1] - b[1]) / (2 * h)
    return g_tr, g_fim


def _away_from_faces(grid, pos, margin=1e-3):
    g = (pos - grid.origin) / grid.voxel_size - 0.5
    frac = g - np.floor(g)
    return ((frac > margin) & (frac < 1 - margin)).all(axis=1)


def _relv(a, b):
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


def _relf(a, b):
    q = a.shape[0]
    return np.linalg.norm((a - b).reshape(q, -1), axis=1) / np.maximum(np.linalg.norm(b.reshape(q, -1), axis=1),
                                                                        1e-300)


# ── A10: indexing, bit-exact ────────────────────────────────────────
def test_locate_vs_reference_golden(g_small, models):
    grid = F.GridConfig(g_small["origin"], g_small["voxel_size"][0], g_small["dims"])
    f = F.Field.build(g_small["points"][:10], grid, models["quad"], "trace")
    pos = g_small["positions"]
    near = f.locate(pos, "nearest")
    ref_n = g_small["nearest_index"]
    assert np.array_equal(near["status"] == 1, ref_n < 0)
    assert np.array_equal(near["index"][:, 0], np.where(ref_n < 0, -1, ref_n))
    assert np.all(near["index"][:, 1:] == -1) and np.all(near["weight"][ref_n >= 0, 0] == 1.0)
    tri = f.locate(pos, "trilinear")
    ref_t = g_small["trilinear_idx_w"]
    out = np.isnan(ref_t[:, 0])
    assert np.array_equal(tri["status"] == 1, out)
    assert np.array_equal(tri["index"][~out].astype(np.float64), ref_t[~out, :8])
    assert np.array_equal(tri["weight"][~out], ref_t[~out, 8:])  # bit-identical weights
    assert np.all(tri["index"][out] == -1) and np.all(tri["weight"][out] == 0)


def _edge_positions(grid, rng, n_random=2000):
    c = grid.centers()
    lo, hi = grid.origin, grid.origin + grid.extent
    pts = [c[0], c[-1], lo, hi, np.nextafter(lo, -np.inf), np.nextafter(hi, np.inf), np.nextafter(hi, -np.inf),
           np.nextafter(c[-1], np.inf), np.nextafter(c[-1], -np.inf), np.nextafter(c[0], -np.inf)]
    pts += list(c[rng.choice(len(c), 200)])                                   # exact centres
    faces = grid.origin + rng.integers(0, grid.dims + 1, size=(200, 3)) * grid.voxel_size  # cell faces / corners
    pts += list(faces)
    for a in range(3):  # one coordinate on the first / last centre or the box face, the others random
        for val in (c[0][a], c[-1][a], lo[a], hi[a], np.nextafter(c[-1][a], np.inf)):
            p = rng.uniform(lo, hi, size=(20, 3))
            p[:, a] = val
            pts += list(p)
    pts += list(rng.uniform(lo - grid.voxel_size, hi + grid.voxel_size, size=(n_random, 3)))
    return np.ascontiguousarray(np.array(pts))


@pytest.mark.parametrize("cfg", ["config1", "config2"])
def test_locate_edges_vs_oracle(oracle, models, cfg):
    w = getattr(scenes, cfg)(0)
    grid = F.GridConfig(*w.grid)
    f = F.Field.build(np.zeros((0, 3)), grid, models["quad"], "trace")
    pos = _edge_positions(grid, np.random.default_rng(5))
    near = f.locate(pos, "nearest")
    tri = f.locate(pos, "trilinear")
    for i, p in enumerate(pos):
        ni = oracle.locate_nearest(grid.origin, grid.voxel_size, grid.dims, p)
        assert near["index"][i, 0] == ni and (near["status"][i] == 1) == (ni < 0), (i, p)
        r = oracle.trilinear(grid.origin, grid.voxel_size, grid.dims, p)
        if r is None:
            assert tri["status"][i] == 1, (i, p)
        else:
            assert tri["status"][i] == 0, (i, p)
            assert np.array_equal(tri["index"][i], r[0]) and np.array_equal(tri["weight"][i], r[1]), (i, p)
    # the query kernels report the same statuses
    q = f.query_batch(pos, axes=np.tile([0.0, 0.0, 1.0], (len(pos), 1)), outputs=("trace",), mode="trilinear",
                      to_numpy=True)
    assert np.array_equal(q["in_field"], tri["status"] == 0)


# ── A14: query_factor ───────────────────────────────────────────────
def test_query_factor_vs_reference(g_small, models):
    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "query_factor.npz"))
    grid = F.GridConfig(g_small["origin"], g_small["voxel_size"][0], g_small["dims"])
    for name, model, kind in (("quad_info", models["quad"], "info"), ("gp30_trace", models["gp30"], "trace")):
        f = F.Field.build(g_small["points"], grid, model, kind, exact=name == "quad_info")
        for mode in ("nearest", "trilinear"):
            ref, ok = g[f"{name}_{mode}"], g[f"ok_{name}_{mode}"]
            for i, p in enumerate(g_small["positions"]):
                if not ok[i]:
                    with pytest.raises(F.OutOfField):
                        f.query_factor(p, mode)
                    continue
                mine = np.asarray(f.query_factor(p, mode)).reshape(-1)
                if name == "quad_info":  # EXACT build: identical rows, identical blend
                    assert np.array_equal(mine, ref[i]), (mode, i)
                else:
                    assert np.linalg.norm(mine - ref[i]) <= TRACE_TOL * np.linalg.norm(ref[i]), (mode, i)


# ── config 1: every query ───────────────────────────────────────────
@pytest.mark.parametrize("mname", ["gp70", "quad"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_config1_all_queries_with_gradients(oracle, models, mname, kind):
    w = scenes.config1(1000)
    grid = F.GridConfig(*w.grid)
    m = models[mname]
    f = F.Field.build(w.points, grid, m, kind)
    res = f.query_batch(w.positions, rotations=w.rotations, outputs=("trace", "full") if kind == "info" else ("trace",),
                        grad=True, to_numpy=True)
    rows = oracle_field(oracle, m, grid.centers(), w.points, kind)  # the oracle's own full-grid build
    slots = np.arange(grid.voxel_count, dtype=np.int32)
    full = kind == "info"
    rt, rf, st = _oracle_query(oracle, slots, rows, grid, m, kind, w.positions, w.rotations, full)
    assert np.array_equal(res["in_field"], st == 0) and res["in_field"].all()
    et = _relv(res["trace"], rt)
    print(f"config1 {mname} {kind}: 1000 queries trace rel {et.max():.2e}", end="")
    assert et.max() <= Q_TOL
    if full:
        ef = _relf(res["fim"], rf)
        print(f", 6x6 relF {ef.max():.2e}", end="")
        assert ef.max() <= Q_TOL
    keep = _away_from_faces(grid, w.positions)
    assert keep.sum() >= 950
    g_tr, g_fim = _fd(oracle, slots, rows, grid, m, kind, w.positions[keep], w.rotations[keep], full)
    eg = np.linalg.norm(res["trace_grad"][keep] - g_tr, axis=1) / np.linalg.norm(g_tr, axis=1)
    print(f", trace grad {eg.max():.2e} ({keep.sum()} FD)", end="")
    assert eg.max() <= Q_TOL
    if full:
        egf = _relf(res["fim_grad"][keep], g_fim)
        print(f", 6x6 grad {egf.max():.2e}", end="")
        assert egf.max() <= Q_TOL
    print()


# ── config 2: >= 1 000 random + >= 1 000 boundary voxels ─────────────
def _config2_voxels(grid, n_random=1000, n_boundary=1000, seed=9):
    rng = np.random.default_rng(seed)
    nx, ny, nz = (int(d) for d in grid.dims)
    idx3 = grid.index3_of(np.arange(grid.voxel_count))
    on_face = ((idx3 == 0) | (idx3 == grid.dims - 1)).any(axis=1)
    face_lin = np.nonzero(on_face)[0]
    corners = np.array([[i, j, k] for i in (0, nx - 1) for j in (0, ny - 1) for k in (0, nz - 1)])
    lin = np.concatenate([rng.choice(np.nonzero(~on_face)[0], n_random, replace=False),
                          rng.choice(face_lin, n_boundary, replace=False), grid.linear_index(corners)])
    return np.unique(lin)


@pytest.mark.parametrize("mname", ["gp70", "quad"])
@pytest.mark.parametrize("kind", ["info", "trace"])
def test_config2_build_2000_voxels(oracle, models, mname, kind):
    w = scenes.config2(0)
    grid = F.GridConfig(*w.grid)
    lin = _config2_voxels(grid)
    assert lin.size >= 2000
    idx3 = grid.index3_of(lin)
    cen = grid.center_of(idx3)
    m = models[mname]
    s64, _ = FD.build_rows(torch.tensor(w.points, device=DEV), m, kind == "trace", 1.0, torch.device(DEV),
                           centers=torch.tensor(cen, device=DEV))
    fld = FD.Field(grid, m, kind, 1.0, s64, None, idx3.astype(np.int32), dense=False)
    ref = oracle_field(oracle, m, cen, w.points, kind)
    err = _err(kind, fld.factors, ref)
    print(f"config2 {mname} {kind}: {lin.size} voxels, max err {err.max():.2e}")
    assert err.max() <= (1e-12 if mname == "quad" else _tol(kind))
    # the dense grid build produces the same rows (explicit-centre and grid modes agree)
    if mname == "gp70" and kind == "info":
        dense = F.Field.build(w.points, grid, m, kind)
        rows = torch.as_tensor(grid.internal_index(idx3), device=DEV)
        assert torch.equal(dense.storage["f64"][rows], s64)


def test_config2_10k_queries_and_1k_gradients(oracle, models):
    """Query parity on the field's own rows: the GPU-built GP-70 info field's reference-layout
    rows (FP64) go through the oracle's FP64 query; the GPU queries stream the FP32 copy."""
    w = scenes.config2(10000)
    grid = F.GridConfig(*w.grid)
    m = models["gp70"]
    f = F.Field.build(w.points, grid, m, "info")
    res = f.query_batch(w.positions, rotations=w.rotations, outputs=("trace", "full"), grad=True, to_numpy=True)
    loc = f.locate(w.positions, "trilinear")
    need = np.unique(loc["index"][loc["index"] >= 0])
    rows = f.slots[need]
    ref_rows = f.export_reference(rows).cpu().numpy()
    slots = np.full(grid.voxel_count, -1, np.int32)
    slots[need] = np.arange(need.size, dtype=np.int32)
    rt, rf, st = _oracle_query(oracle, slots, ref_rows, grid, m, "info", w.positions, w.rotations, True)
    assert np.array_equal(res["in_field"], st == 0)
    et, ef = _relv(res["trace"], rt), _relf(res["fim"], rf)
    print(f"config2 10k queries: trace {et.max():.2e}, 6x6 {ef.max():.2e}", end="")
    assert et.max() <= Q_TOL and ef.max() <= Q_TOL
    keep = np.nonzero(_away_from_faces(grid, w.positions))[0][:1000]
    g_tr, g_fim = _fd(oracle, slots, ref_rows, grid, m, "info", w.positions[keep], w.rotations[keep], True)
    eg = np.linalg.norm(res["trace_grad"][keep] - g_tr, axis=1) / np.linalg.norm(g_tr, axis=1)
    egf = _relf(res["fim_grad"][keep], g_fim)
    print(f", {keep.size} FD gradients: trace {eg.max():.2e}, 6x6 {egf.max():.2e}")
    assert eg.max() <= Q_TOL and egf.max() <= Q_TOL
    # nearest mode on the same batch (one corner: no blending to average the copy's rounding)
    rn = f.query_batch(w.positions, rotations=w.rotations, outputs=("trace", "full"), mode="nearest", to_numpy=True)
    locn = f.locate(w.positions, "nearest")
    needn = np.unique(locn["index"][locn["index"] >= 0])
    sl = np.full(grid.voxel_count, -1, np.int32)
    sl[needn] = np.arange(needn.size, dtype=np.int32)
    rr = f.export_reference(f.slots[needn]).cpu().numpy()
    ax = np.ascontiguousarray(w.rotations[:, :, 2])
    tn, stn = oracle.metric_batch(sl, rr, grid.origin, grid.voxel_size, grid.dims, w.positions, ax, oracle_model(m),
                                  "trace", False, False)
    fn, _ = oracle.query_fim_batch(sl, rr, grid.origin, grid.voxel_size, grid.dims, w.positions, ax, oracle_model(m),
                                   False)
    print(f"config2 10k nearest: trace {_relv(rn['trace'], tn).max():.2e}, 6x6 {_relf(rn['fim'], fn).max():.2e}")
    assert np.array_equal(rn["in_field"], stn == 0) and _relv(rn["trace"], tn).max() <= Q_TOL
    assert _relf(rn["fim"], fn).max() <= Q_TOL


@pytest.mark.parametrize("mode", ["nearest", "trilinear"])
def test_config2_trace_field_10k_queries(oracle, models, mode):
    """GP-70 TRACE field on config 2 (the FP64 master is the query operand), 10 000 queries."""
    w = scenes.config2(10000)
    grid = F.GridConfig(*w.grid)
    m = models["gp70"]
    f = F.Field.build(w.points, grid, m, "trace")
    res = f.query_batch(w.positions, rotations=w.rotations, outputs=("trace",), grad=mode == "trilinear",
                        mode=mode, to_numpy=True)
    loc = f.locate(w.positions, mode)
    need = np.unique(loc["index"][loc["index"] >= 0])
    slots = np.full(grid.voxel_count, -1, np.int32)
    slots[need] = np.arange(need.size, dtype=np.int32)
    rows = f.export_reference(f.slots[need]).cpu().numpy()
    ax = np.ascontiguousarray(w.rotations[:, :, 2])
    tr, st = oracle.metric_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, w.positions, ax,
                                 oracle_model(m), "trace", True, mode == "trilinear")
    e = _relv(res["trace"], tr)
    print(f"config2 trace field {mode}: 10k queries trace rel {e.max():.2e}")
    assert np.array_equal(res["in_field"], st == 0) and e.max() <= Q_TOL
    if mode == "trilinear":
        keep = np.nonzero(_away_from_faces(grid, w.positions))[0][:500]
        g_tr, _ = _fd(oracle, slots, rows, grid, m, "trace", w.positions[keep], w.rotations[keep], False)
        eg = np.linalg.norm(res["trace_grad"][keep] - g_tr, axis=1) / np.linalg.norm(g_tr, axis=1)
        assert eg.max() <= Q_TOL


# ── config 3: 10 000 poses, masks bit-exact ─────────────────────────
def test_config3_10k_poses_masks_bit_exact(oracle):
    w = scenes.config3(10000)
    cam = F.PinholeCamera.from_fov()
    r = torch.tensor(w.rotations.reshape(-1, 9), device=DEV)
    t = torch.tensor(w.positions, device=DEV)
    p = torch.tensor(w.points, device=DEV)
    mask = torch.zeros((10000, w.points.shape[0]), dtype=torch.uint8, device=DEV)
    out = F.exact_pose_fim_batch_device(r, t, p, cam, mask=mask).cpu().numpy().reshape(-1, 6, 6)
    om = oracle.pc_mask(w.rotations, w.positions, w.points, cam.as_tuple())
    assert np.array_equal(mask.cpu().numpy().astype(bool), om)  # 2e8 pairs
    ref = oracle.exact_fim_batch(w.rotations, w.positions, w.points, cam.as_tuple())
    e = _relf(out, ref)
    print(f"config3 10k poses: visible fraction {om.mean():.4f}, 6x6 relF {e.max():.2e}")
    assert e.max() <= 1e-4


# ── config 4: >= 256 voxels per kind incl. every slab seam ──────────
def _seam_rows(V):
    seams = sorted({slab_range(V, n, r)[0] for n in (2, 4, 8) for r in range(1, n)})
    return seams


@pytest.mark.parametrize("mname", ["gp70", "quad"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_config4_256_voxels_with_slab_seams(oracle, models, mname, kind):
    """Seam voxels (both sides of every 2/4/8-way split) are built in grid/slab mode exactly as
    the ranks build them; random voxels through the explicit-centre mode."""
    w = scenes.config4(kind, n_points=0)
    pts = scenes.config4(kind).points
    grid = F.GridConfig(*w.grid)
    V = grid.voxel_count
    m = models[mname]
    dev = torch.device(DEV)
    P = torch.tensor(pts, device=dev)
    seams = _seam_rows(V)
    got, idx3 = [], []
    for s in seams:  # rows [s-2, s+2): two voxels on each side of the seam, as two slab launches
        for b0, b1 in ((s - 2, s), (s, s + 2)):
            r64, _ = FD.build_rows(P, m, kind == "trace", 1.0, dev, grid=grid, v_begin=b0, v_end=b1)
            got.append(r64)
            idx3.append(grid.index3_of_internal(np.arange(b0, b1)))
    n_seam = sum(g.shape[0] for g in got)
    rng = np.random.default_rng(13)
    n_rand = 256 - n_seam
    i3r = grid.index3_of(rng.choice(V, n_rand, replace=False))
    r64, _ = FD.build_rows(P, m, kind == "trace", 1.0, dev, centers=torch.tensor(grid.center_of(i3r), device=dev))
    got.append(r64)
    idx3.append(i3r)
    idx3 = np.vstack(idx3)
    s64 = torch.cat(got)
    assert s64.shape[0] >= 256
    fld = FD.Field(grid, m, kind, 1.0, s64, None, idx3.astype(np.int32), dense=False)
    cen = grid.center_of(idx3)
    ref = oracle_field(oracle, m, cen, pts, kind)
    err = _err(kind, fld.factors, ref)
    print(f"config4 {mname} {kind}: {s64.shape[0]} voxels ({n_seam} on {len(seams)} slab seams), max err "
          f"{err.max():.2e}")
    assert err.max() <= (1e-12 if mname == "quad" else _tol(kind))


# ── config 5: >= 1 000 values + 64 FD gradients ─────────────────────
def test_config5_1000_queries_64_gradients(oracle, models):
    w = scenes.config4("info", n_points=0)
    pts = scenes.config4("info").points
    grid = F.GridConfig(*w.grid)
    rng = np.random.default_rng(4)
    pos, rot = scenes.bspline_trajectory_batch(rng, 20)  # 20 x 64 poses of the config-5 stream
    m = models["gp70"]
    dev = torch.device(DEV)
    # a cropped GPU field: the voxels these queries touch, built in explicit-centre mode
    tmp = F.Field.build(np.zeros((0, 3)), grid, m, "trace")
    loc = tmp.locate(pos, "trilinear")
    inside = loc["status"] == 0
    pos, rot = pos[inside], rot[inside]
    assert pos.shape[0] >= 1000
    need = np.unique(loc["index"][inside][loc["index"][inside] >= 0])
    cen = grid.centers()[need]
    s64, s32 = FD.build_rows(torch.tensor(pts, device=dev), m, False, 1.0, dev, centers=torch.tensor(cen, device=dev))
    fld = FD.Field(grid, m, "info", 1.0, s64, s32, grid.index3_of(need).astype(np.int32), dense=False)
    res = fld.query_batch(pos, rotations=rot, outputs=("trace", "full"), grad=True, to_numpy=True)
    slots = np.full(grid.voxel_count, -1, np.int32)
    slots[need] = np.arange(need.size, dtype=np.int32)
    rows = fld.factors  # this field's own rows, FP64 reference layout
    rt, rf, st = _oracle_query(oracle, slots, rows, grid, m, "info", pos, rot, True)
    assert np.array_equal(res["in_field"], st == 0) and res["in_field"].all()
    et, ef = _relv(res["trace"], rt), _relf(res["fim"], rf)
    keep = np.nonzero(_away_from_faces(grid, pos))[0][:64]
    assert keep.size == 64
    g_tr, g_fim = _fd(oracle, slots, rows, grid, m, "info", pos[keep], rot[keep], True)
    eg = np.linalg.norm(res["trace_grad"][keep] - g_tr, axis=1) / np.linalg.norm(g_tr, axis=1)
    egf = _relf(res["fim_grad"][keep], g_fim)
    print(f"config5 {pos.shape[0]} queries: trace {et.max():.2e}, 6x6 {ef.max():.2e}; 64 FD grads: trace "
          f"{eg.max():.2e}, 6x6 {egf.max():.2e}")
    assert et.max() <= Q_TOL and ef.max() <= Q_TOL and eg.max() <= Q_TOL and egf.max() <= Q_TOL
    # end to end on 48 voxels' worth of queries: the oracle's own rows for the first batch
    q0 = slice(0, 64)
    need0 = np.unique(loc["index"][inside][q0][loc["index"][inside][q0] >= 0])
    rows0 = oracle_field(oracle, m, grid.centers()[need0], pts, "info")
    sl0 = np.full(grid.voxel_count, -1, np.int32)
    sl0[need0] = np.arange(need0.size, dtype=np.int32)
    rt0, rf0, _ = _oracle_query(oracle, sl0, rows0, grid, m, "info", pos[q0], rot[q0], True)
    assert _relv(res["trace"][q0], rt0).max() <= Q_TOL and _relf(res["fim"][q0], rf0).max() <= Q_TOL


# ── A16: planner variant pc_metric_yaw_batch / ExactInfoRepr ────────
def test_pc_metric_yaw_vs_reference_golden():
    import os

    from paper_2008_03324_b200.planner import ExactInfoRepr, R_CAM_MOUNT

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "pc_yaw.npz"))
    assert np.array_equal(g["r_base"], R_CAM_MOUNT)
    rep = ExactInfoRepr(g["points"])
    for metric in ("det", "lmin", "trace"):
        v, ok = rep.metric_batch(g["positions"], g["yaws"], metric)
        ref = g[metric]
        assert ok.all()
        scale = np.abs(ref).max()
        big = np.abs(ref) > 1e-3 * scale
        print(f"pc_metric_yaw {metric}: rel {_relv(v, ref)[big].max():.2e}, vs batch scale "
              f"{(np.abs(v - ref) / scale).max():.2e}")
        # det / lambda_min of an ill-conditioned 6x6 amplify the FP32 accumulation's relative
        # error by its condition number: compared against the batch scale like the field's
        # det / lmin queries (test_gpu_query.py); the trace per value
        assert (np.abs(v - ref) / scale).max() <= Q_TOL
        if metric == "trace":
            assert _relv(v, ref).max() <= Q_TOL
    cam = F.PinholeCamera.from_fov()
    v7 = F.pc_metric_yaw_batch(g["positions"], g["yaws"], g["points"], cam, 0.7, R_CAM_MOUNT, "trace")
    assert _relv(v7, g["trace_sigma07"]).max() <= 1e-5
    # masks of the yaw poses (incl. landmarks on the image borders) bit-exact
    dev = torch.device(DEV)
    q, n = g["positions"].shape[0], g["points"].shape[0]
    mask = torch.zeros((q, n), dtype=torch.uint8, device=dev)
    F.pc_metric_yaw_batch_device(torch.tensor(g["positions"], device=dev), g["yaws"],
                                 torch.tensor(g["points"], device=dev), cam, 1.0, R_CAM_MOUNT, "trace", mask=mask)
    assert np.array_equal(mask.cpu().numpy().astype(bool), g["visible_kernel"])


def test_pc_metric_yaw_config3_scale(oracle):
    """10 000 yaw poses against the config-2 room: masks bit-exact, det / trace vs the oracle."""
    from paper_2008_03324_b200.planner import R_CAM_MOUNT

    w = scenes.config3(10000)
    rng = np.random.default_rng(6)
    yaws = rng.uniform(-np.pi, np.pi, 10000)
    cam = F.PinholeCamera.from_fov()
    dev = torch.device(DEV)
    mask = torch.zeros((10000, w.points.shape[0]), dtype=torch.uint8, device=dev)
    fim = torch.empty((10000, 36), dtype=torch.float64, device=dev)
    vals = F.pc_metric_yaw_batch_device(torch.tensor(w.positions, device=dev), yaws, torch.tensor(w.points, device=dev),
                                        cam, 1.0, R_CAM_MOUNT, "det", fim=fim, mask=mask).cpu().numpy()
    c, s = np.cos(yaws), np.sin(yaws)
    b = R_CAM_MOUNT
    rots = np.empty((10000, 3, 3))
    for col in range(3):  # kernels.py:615-621, numpy rounds each product / sum like numba
        rots[:, 0, col] = c * b[0, col] - s * b[1, col]
        rots[:, 1, col] = s * b[0, col] + c * b[1, col]
        rots[:, 2, col] = b[2, col]
    om = oracle.pc_mask(rots, w.positions, w.points, cam.as_tuple())
    assert np.array_equal(mask.cpu().numpy().astype(bool), om)
    ref = oracle.exact_fim_batch(rots, w.positions, w.points, cam.as_tuple())
    assert _relf(fim.cpu().numpy().reshape(-1, 6, 6), ref).max() <= 1e-4
    rdet = np.array([oracle.metric_of(f, "det") for f in ref])
    scale = np.abs(rdet).max()
    assert (np.abs(vals - rdet) / scale).max() <= Q_TOL

"""GPU query parity (fif_query through the C ABI) vs the reference and the oracle.

Values: trace relative <= 1e-4, 6x6 relative Frobenius <= 1e-4; det / lmin relative to
the batch scale <= 1e-4; status bit-exact.  Gradients (new capability):
<= 1e-4 relative to a central finite difference (h = 1e-6) of the FP64 oracle query,
t' = t + dt, R' = exp(dtheta^) R.
"""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD
from paper_2008_03324_b200.geometry import so3_exp
from tests._helpers import models_from_golden, oracle_model

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def models(g_models):
    return models_from_golden(g_models)


@pytest.fixture(scope="module")
def small_grid(g_small):
    return F.GridConfig(g_small["origin"], g_small["voxel_size"][0], g_small["dims"])


def field_from_reference(grid, model, kind, factors):
    """A device Field holding exactly the reference's rows (x-major, all voxels)."""
    s64 = torch.tensor(FD._from_reference_rows(factors, model, kind), device="cuda")
    s32 = s64.float() if isinstance(model, F.GpVisibility) else None
    occ = grid.index3_of(np.arange(grid.voxel_count)).astype(np.int32)
    return FD.Field(grid, model, kind, 1.0, s64, s32, occ, dense=False)


def rel(a, b):
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


@pytest.mark.parametrize("mname", ["quad", "gp30", "gp70"])
@pytest.mark.parametrize("kind", ["trace", "info"])
@pytest.mark.parametrize("mode", ["nearest", "trilinear"])
@pytest.mark.parametrize("source", ["reference_field", "gpu_build"])
def test_queries_vs_reference(g_small, models, small_grid, mname, kind, mode, source):
    m = models[mname]
    if source == "reference_field":
        f = field_from_reference(small_grid, m, kind, g_small[f"factors_{mname}_{kind}"])
    else:
        f = F.Field.build(g_small["points"], small_grid, m, kind)
    pos, rots = g_small["positions"], g_small["rotations"]
    axes = np.ascontiguousarray(rots[:, :, 2])
    ok_ref = g_small[f"ok_{mname}_{kind}_{mode}"]
    vals, ok = f.metric_axis_batch(pos, axes, "trace", mode)
    assert np.array_equal(ok, ok_ref)
    ref = g_small[f"trace_{mname}_{kind}_{mode}"]
    assert rel(vals, ref)[ok_ref].max() <= TOL
    assert np.all(vals[~ok_ref] == 0)
    if kind == "info":
        fims, ok2 = f.query_fim_batch(pos, rots, mode)
        assert np.array_equal(ok2, ok_ref)
        rf = g_small[f"fim_{mname}_{mode}"]
        e = np.linalg.norm((fims - rf).reshape(len(pos), -1), axis=1) / np.maximum(
            np.linalg.norm(rf.reshape(len(pos), -1), axis=1), 1e-300)
        assert e[ok_ref].max() <= TOL
        assert np.allclose(fims, np.transpose(fims, (0, 2, 1)))
        for metric in ("det", "lmin"):
            mv, _ = f.metric_axis_batch(pos, axes, metric, mode)
            rm = g_small[f"{metric}_{mname}_{mode}"]
            assert (np.abs(mv - rm)[ok_ref].max() / np.abs(rm[ok_ref]).max()) <= TOL


def test_single_pose_api_errors(g_small, models, small_grid):
    f = F.Field.build(g_small["points"], small_grid, models["quad"], "info")
    ft = F.Field.build(g_small["points"], small_grid, models["quad"], "trace")
    inside = F.Pose(F.random_rotation(np.random.default_rng(1)), small_grid.center_of([2, 2, 2]) + 0.1)
    outside = F.Pose(np.eye(3), small_grid.origin - 1.0)
    assert f.query_fim(inside, "trilinear").shape == (6, 6)
    with pytest.raises(F.OutOfField):
        f.query_fim(outside)
    with pytest.raises(F.OutOfField):
        f.query_metric(outside, "trace")
    with pytest.raises(F.WrongFactorKind):
        ft.query_fim(inside)
    with pytest.raises(F.WrongFactorKind):
        ft.query_metric(inside, "det")
    with pytest.raises(ValueError):
        f.query_fim(inside, "cubic")
    assert ft.query_metric(inside, "trace", "trilinear") == pytest.approx(
        f.query_metric(inside, "trace", "trilinear"), rel=1e-9)  # trace consistency


def _fd_queries(oracle, factors, grid, model, kind, pos, rots, h=1e-6):
    """Central FD of the oracle's trilinear trace (and 6x6 for info) w.r.t. [t; theta]."""
    slots = np.arange(grid.voxel_count, dtype=np.int32)
    om = oracle_model(model)

    def ev(p, r):
        ax = np.ascontiguousarray(r[:, :, 2])
        tr, st = oracle.metric_batch(slots, factors, grid.origin, grid.voxel_size, grid.dims, p, ax, om, "trace",
                                     kind == "trace", True)
        fim = None
        if kind == "info":
            fim, _ = oracle.query_fim_batch(slots, factors, grid.origin, grid.voxel_size, grid.dims, p, ax, om, True)
        return tr, fim, st

    q = pos.shape[0]
    g_tr = np.zeros((q, 6))
    g_fim = np.zeros((q, 6, 6, 6)) if kind == "info" else None
    for j in range(6):
        if j < 3:
            d = np.zeros(3)
            d[j] = h
            a, b = ev(pos + d, rots), ev(pos - d, rots)
        else:
            w = np.zeros(3)
            w[j - 3] = h
            Rp, Rm = so3_exp(w), so3_exp(-w)
            a = ev(pos, np.einsum("ij,qjk->qik", Rp, rots))
            b = ev(pos, np.einsum("ij,qjk->qik", Rm, rots))
        g_tr[:, j] = (a[0] - b[0]) / (2 * h)
        if kind == "info":
            g_fim[:, j] = (a[1] - b[1]) / (2 * h)
    return g_tr, g_fim


@pytest.mark.parametrize("mname", ["quad", "gp30", "gp70"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_gradients_vs_finite_difference(oracle, g_small, models, small_grid, mname, kind):
    m = models[mname]
    factors = g_small[f"factors_{mname}_{kind}"]
    f = field_from_reference(small_grid, m, kind, factors)
    rng = np.random.default_rng(17)
    c = small_grid.centers()
    pos = rng.uniform(c[0], c[-1], size=(60, 3))
    g = (pos - small_grid.origin) / small_grid.voxel_size - 0.5
    frac = g - np.floor(g)
    pos = pos[((frac > 1e-3) & (frac < 1 - 1e-3)).all(axis=1)]  # >= 2h away from cell faces
    rots = np.stack([F.random_rotation(rng) for _ in range(pos.shape[0])])
    outs = ("trace", "full") if kind == "info" else ("trace",)
    for f64 in (True, False):
        dev = torch.device("cuda")
        res = f.query_device(torch.tensor(pos, device=dev), torch.tensor(np.ascontiguousarray(rots[:, :, 2]), device=dev),
                             "trilinear", trace=True, full=kind == "info", grad=True, field_f64=f64)
        g_tr_fd, g_fim_fd = _fd_queries(oracle, factors, small_grid, m, kind, pos,
                                        rots)
        g_tr = res["trace_grad"].cpu().numpy()
        err = np.linalg.norm(g_tr - g_tr_fd, axis=1) / np.linalg.norm(g_tr_fd, axis=1)
        print(f"[grad {mname} {kind} f64={f64}] trace grad {err.max():.2e}", end="")
        tol = TOL  # the north_star's 1e-4, FP32 and FP64 query copies alike
        assert err.max() <= tol, (f64, err.max())
        if kind == "info":
            g_f = res["fim_grad"].cpu().numpy().reshape(-1, 6, 6, 6)
            e2 = np.linalg.norm((g_f - g_fim_fd).reshape(len(pos), -1), axis=1) / np.linalg.norm(
                g_fim_fd.reshape(len(pos), -1), axis=1)
            print(f" 6x6 grad {e2.max():.2e}", end="")
            assert e2.max() <= tol, (f64, e2.max())
        print()


def test_config2_queries_end_to_end(oracle, models):
    """GPU-built config-2 field, 64 trilinear queries with gradient, vs the oracle on a cropped field."""
    from paper_2008_03324_b200 import scenes
    from tests._helpers import oracle_field

    w = scenes.config2(64)
    grid = F.GridConfig(*w.grid)
    for mname in ("quad", "gp70"):
        m = models[mname]
        f = F.Field.build(w.points, grid, m, "info")
        res = f.query_batch(w.positions, rotations=w.rotations, outputs=("trace", "full"), grad=True,
                            to_numpy=True)
        need = sorted({int(i) for p in w.positions for i in oracle.trilinear(grid.origin, grid.voxel_size,
                                                                            grid.dims, p)[0]})
        need = np.array(need)
        rows = oracle_field(oracle, m, grid.centers()[need], w.points, "info")
        slots = np.full(grid.voxel_count, -1, np.int32)
        slots[need] = np.arange(len(need), dtype=np.int32)
        ax = np.ascontiguousarray(w.rotations[:, :, 2])
        rt, st = oracle.metric_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, w.positions, ax,
                                     oracle_model(m), "trace", False, True)
        rf, _ = oracle.query_fim_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, w.positions, ax,
                                       oracle_model(m), True)
        assert np.array_equal(res["in_field"], st == 0)
        assert rel(res["trace"], rt).max() <= TOL
        e = np.linalg.norm((res["fim"] - rf).reshape(64, -1), axis=1) / np.linalg.norm(rf.reshape(64, -1), axis=1)
        assert e.max() <= TOL
        assert np.isfinite(res["fim_grad"]).all()


def test_factorization_exact_at_voxel_centres(models):
    """at a voxel centre the field FIM equals sum_i v_model(theta_i) I_i
    (1e-9 for the FP64 quad build; GP builds use FP32/TF32 per-pair arithmetic, so the
    bar is the query tolerance's 10x-tighter 1e-5)."""
    rng = np.random.default_rng(4)
    pts = rng.uniform([-3, -3, 0], [3, 3, 3], size=(150, 3))
    grid = F.GridConfig(np.array([-1.0, -1.0, 0.5]), 0.5, np.array([4, 4, 3]))
    for mname in ("quad", "gp30"):
        m = models[mname]
        f = F.Field.build(pts, grid, m, "info")
        for idx in ([1, 1, 1], [2, 3, 0]):
            c = grid.center_of(idx)
            R = F.random_rotation(rng)
            got = f.query_fim(F.Pose(R, c), "nearest")
            vr = m.rotation_vector(R)
            vp = m.position_vectors(c, pts)
            direct = sum(float(vr @ vp[i]) * F.landmark_fim(c, pts[i]) for i in range(len(pts)))
            tol = 1e-9 if mname == "quad" else 1e-5
            assert np.linalg.norm(got - direct) <= tol * np.linalg.norm(direct)


@pytest.mark.parametrize("mname", ["quad", "gp70"])
@pytest.mark.parametrize("metric", ["det", "lmin"])
def test_metric_gradients_vs_finite_difference(oracle, g_small, models, small_grid, mname, metric):
    """d det / d lambda_min w.r.t. [t; theta] against central FD of
    the oracle's blended metric (kernels.py:1429-1472), h = 1e-6."""
    m = models[mname]
    factors = g_small[f"factors_{mname}_info"]
    f = field_from_reference(small_grid, m, "info", factors)
    rng = np.random.default_rng(23)
    c = small_grid.centers()
    pos = rng.uniform(c[0], c[-1], size=(60, 3))
    g = (pos - small_grid.origin) / small_grid.voxel_size - 0.5
    frac = g - np.floor(g)
    pos = pos[((frac > 1e-3) & (frac < 1 - 1e-3)).all(axis=1)]
    rots = np.stack([F.random_rotation(rng) for _ in range(pos.shape[0])])
    slots = np.arange(small_grid.voxel_count, dtype=np.int32)
    om = oracle_model(m)

    def ev(p, r):
        v, _ = oracle.metric_batch(slots, factors, small_grid.origin, small_grid.voxel_size, small_grid.dims, p,
                                   np.ascontiguousarray(r[:, :, 2]), om, metric, False, True)
        return v

    h = 1e-6
    fd = np.zeros((pos.shape[0], 6))
    for j in range(6):
        if j < 3:
            d = np.zeros(3)
            d[j] = h
            fd[:, j] = (ev(pos + d, rots) - ev(pos - d, rots)) / (2 * h)
        else:
            w = np.zeros(3)
            w[j - 3] = h
            fd[:, j] = (ev(pos, np.einsum("ij,qjk->qik", so3_exp(w), rots)) -
                        ev(pos, np.einsum("ij,qjk->qik", so3_exp(-w), rots))) / (2 * h)
    val = ev(pos, rots)
    for f64 in (True, False):
        dev = torch.device("cuda")
        res = f.query_device(torch.tensor(pos, device=dev), torch.tensor(np.ascontiguousarray(rots[:, :, 2]), device=dev),
                             "trilinear", trace=False, grad=True, det=metric == "det", lmin=metric == "lmin",
                             field_f64=f64)
        mine_v = res[metric].cpu().numpy()
        mine_g = res[f"{metric}_grad"].cpu().numpy()
        tol = TOL  # the north_star's 1e-4, FP32 and FP64 query copies alike
        ev_err = np.abs(mine_v - val) / np.abs(val)
        assert ev_err.max() <= tol, (f64, ev_err.max())
        err = np.linalg.norm(mine_g - fd, axis=1) / np.linalg.norm(fd, axis=1)
        print(f"[metric grad {mname} {metric} f64={f64}] value {ev_err.max():.2e} grad {err.max():.2e}")
        assert err.max() <= tol, (f64, err.max())


@pytest.mark.parametrize("ns", [7, 150, 220])
def test_gp_query_other_sizes(oracle, ns):
    """GP query path at N_s = 7 (one k-chunk), 150 (kinv too large for the DMMA prep's
    shared-memory tile: SIMT prep) and 220 (three warps per voxel in the info build) on a
    GPU-built field vs the oracle."""
    from tests._helpers import oracle_field

    m = F.build_gp_model(ns)
    rng = np.random.default_rng(ns)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(250, 3))
    grid = F.GridConfig(np.array([-1.0, -1.0, 0.25]), 0.5, np.array([4, 4, 3]))
    f = F.Field.build(pts, grid, m, "info")
    c = grid.centers()
    pos = rng.uniform(c[0], c[-1], size=(50, 3))
    rots = np.stack([F.random_rotation(rng) for _ in range(50)])
    res = f.query_batch(pos, rotations=rots, outputs=("trace", "full"), grad=True, to_numpy=True)
    rows = oracle_field(oracle, m, c, pts, "info")
    slots = np.arange(grid.voxel_count, dtype=np.int32)
    ax = np.ascontiguousarray(rots[:, :, 2])
    rt, st = oracle.metric_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, pos, ax, oracle_model(m),
                                 "trace", False, True)
    rf, _ = oracle.query_fim_batch(slots, rows, grid.origin, grid.voxel_size, grid.dims, pos, ax, oracle_model(m),
                                   True)
    assert np.array_equal(res["in_field"], st == 0)
    assert rel(res["trace"], rt).max() <= TOL
    e = np.linalg.norm((res["fim"] - rf).reshape(50, -1), axis=1) / np.linalg.norm(rf.reshape(50, -1), axis=1)
    assert e.max() <= TOL


def test_query_graph_matches_direct(g_small, models, small_grid):
    """CUDA-graph-captured fixed-size queries (Field.query_graph) == direct queries."""
    m = models["gp70"]
    f = field_from_reference(small_grid, m, "info", g_small["factors_gp70_info"])
    rng = np.random.default_rng(3)
    c = small_grid.centers()
    qg = f.query_graph(64, "trilinear", outputs=("trace", "full", "det"), grad=True)
    for n in (64, 37):
        pos = rng.uniform(c[0], c[-1], size=(n, 3))
        rots = np.stack([F.random_rotation(rng) for _ in range(n)])
        ax = np.ascontiguousarray(rots[:, :, 2])
        got = {k: v[:n].cpu().numpy() for k, v in qg.run(pos, ax).items()}
        ref = f.query_device(torch.tensor(pos, device="cuda"), torch.tensor(ax, device="cuda"), "trilinear",
                             trace=True, full=True, det=True, grad=True)
        for k in ("trace", "trace_grad", "fim", "fim_grad", "det", "det_grad", "status"):
            assert np.array_equal(got[k], ref[k].cpu().numpy()), k


def test_very_large_batch_is_sliced(g_small, models, small_grid):
    """Batches above the per-call scratch bound run as slices (and in locality order):
    every query's result equals the same query issued alone."""
    m = models["gp30"]
    f = field_from_reference(small_grid, m, "info", g_small["factors_gp30_info"])
    rng = np.random.default_rng(8)
    c = small_grid.centers()
    n = (1 << 21) + 1500
    pos = torch.tensor(rng.uniform(c[0] - 0.3, c[-1] + 0.3, size=(n, 3)), device="cuda")
    ax = torch.nn.functional.normalize(torch.tensor(rng.standard_normal((n, 3)), device="cuda"), dim=1)
    big = f.query_device(pos, ax, "trilinear", trace=True, full=True, grad=True)
    for sl in (slice(0, 700), slice((1 << 21) - 300, (1 << 21) + 300), slice(n - 500, n)):
        small = f.query_device(pos[sl].contiguous(), ax[sl].contiguous(), "trilinear", trace=True, full=True, grad=True)
        for k in ("trace", "trace_grad", "fim", "fim_grad", "status"):
            assert torch.equal(big[k][sl], small[k]), k


def test_slab_fields_answer_their_queries_bit_exactly(models):
    """The device side of slab-routed queries (parallel.py): a rank's slab Field (owned
    z-planes + one halo plane, slots over the global grid) answers the queries routed to
    it exactly like the full field."""
    from paper_2008_03324_b200 import field as FDm
    from paper_2008_03324_b200.parallel import query_owners, slab_rows_range

    rng = np.random.default_rng(21)
    pts = rng.uniform([-3, -3, 0], [3, 3, 3], size=(400, 3))
    grid = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([5, 4, 9]))
    m = models["gp30"]
    full = F.Field.build(pts, grid, m, "info")
    dev = torch.device("cuda")
    pts_dev = torch.tensor(pts, device=dev)
    c = grid.centers()
    pos = rng.uniform(c[0] - 0.3, c[-1] + 0.3, size=(300, 3))
    ax = np.ascontiguousarray(np.stack([F.random_rotation(rng) for _ in range(300)])[:, :, 2])
    for world in (2, 3):
        for mode in ("trilinear", "nearest"):
            owner = query_owners(pos, grid, world, mode == "trilinear")
            for rank in range(world):
                _, _, v0, v1 = slab_rows_range(grid, world, rank)
                s64, s32 = FDm.build_rows(pts_dev, m, False, 1.0, dev, grid=grid, v_begin=v0, v_end=v1)
                occ3 = grid.index3_of_internal(np.arange(v0, v1)).astype(np.int32)
                slab = FDm.Field(grid, m, "info", 1.0, s64, s32, occ3, dense=False)
                sel = owner == rank
                p = torch.tensor(pos[sel], device=dev)
                a = torch.tensor(ax[sel], device=dev)
                got = slab.query_device(p, a, mode, trace=True, full=True, grad=True)
                ref = full.query_device(p, a, mode, trace=True, full=True, grad=True)
                for k in ("trace", "trace_grad", "fim", "fim_grad", "status"):
                    assert torch.equal(got[k], ref[k]), (world, mode, rank, k)


@pytest.mark.parametrize("mode", ["trilinear", "nearest"])
def test_streaming_and_fused_small_paths_agree(g_small, models, small_grid, mode):
    """Batches above 444 queries take the streaming kernels (prep + TMA ring), smaller
    GP batches the fused per-query kernel: the two agree (summation order only) for every
    output, metrics and metric gradients included (this also covers the streaming metric
    kernel variants, which the small-batch tests do not reach)."""
    m = models["gp70"]
    f = field_from_reference(small_grid, m, "info", g_small["factors_gp70_info"])
    rng = np.random.default_rng(41)
    c = small_grid.centers()
    n = 900
    pos = torch.tensor(rng.uniform(c[0] - 0.2, c[-1] + 0.2, size=(n, 3)), device="cuda")
    ax = torch.nn.functional.normalize(torch.tensor(rng.standard_normal((n, 3)), device="cuda"), dim=1)
    kw = dict(trace=True, full=True, det=True, lmin=True, grad=True)
    big = f.query_device(pos, ax, mode, **kw)
    for s in (0, 300, 600):
        small = f.query_device(pos[s:s + 300].contiguous(), ax[s:s + 300].contiguous(), mode, **kw)
        assert torch.equal(small["status"], big["status"][s:s + 300])
        for k in ("trace", "trace_grad", "fim", "fim_grad", "det", "det_grad", "lmin", "lmin_grad"):
            a, b = small[k].cpu().numpy(), big[k][s:s + 300].cpu().numpy()
            scale = np.abs(b).reshape(b.shape[0], -1).max(axis=1) + 1e-300
            err = np.abs(a - b).reshape(a.shape[0], -1).max(axis=1) / scale
            # det / lambda_min amplify the entries' last-bit differences by the 6x6's condition
            tol = 1e-6 if k.startswith(("det", "lmin")) else 1e-9
            assert err.max() <= tol, (k, err.max())

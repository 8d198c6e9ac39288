"""GPU build parity: CUDA path (through the C ABI) vs the reference / oracle.

Tolerances (BASELINE north_star): trace PIF per-voxel relative L2
<= 1e-5; full PIF max-entry |delta| <= 1e-4 x voxel Frobenius norm; quad in
EXACT mode bit-identical; voxel centres bit-exact.
"""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import _lib
from paper_2008_03324_b200 import field as FD
from tests._helpers import info_rel_fro, models_from_golden, oracle_field, reference_order, trace_rel_l2

pytestmark = pytest.mark.gpu
TRACE_TOL, INFO_TOL = 1e-5, 1e-4


@pytest.fixture(scope="module")
def models(g_models):
    return models_from_golden(g_models)


@pytest.fixture(scope="module")
def small_grid(g_small):
    return F.GridConfig(g_small["origin"], g_small["voxel_size"][0], g_small["dims"])


@pytest.mark.parametrize("order", [0, 1])
def test_centers_bit_exact(oracle, small_grid, order):
    dev = torch.device("cuda")
    V = small_grid.voxel_count
    out = torch.empty((V, 3), dtype=torch.float64, device=dev)
    g = _lib.make_grid(small_grid.origin, small_grid.voxel_size, small_grid.dims)
    _lib.check(_lib.load().fif_grid_centers(g, order, 0, V, out.data_ptr(), None), "centers")
    ref = oracle.centers(small_grid.origin, small_grid.voxel_size, small_grid.dims)
    if order == 1:
        ref = ref[np.argsort(small_grid.internal_index(small_grid.index3_of(np.arange(V))))]
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.fixture(params=["t5", "h16", "tf32", "simt"])
def gp_info_kernel(request, monkeypatch):
    """Every GP-info kernel (tcgen05 default, mma.sync FP16-split, TF32x3, FP32 FFMA2 SIMT) must meet parity."""
    monkeypatch.setattr(FD, "GP_INFO_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("mname", ["quad", "gp30", "gp70"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_build_vs_reference_golden(g_small, models, small_grid, mname, kind, gp_info_kernel):
    f = F.Field.build(g_small["points"], small_grid, models[mname], kind)
    mine, ref = reference_order(f), g_small[f"factors_{mname}_{kind}"]
    err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
    assert err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL)
    if mname == "quad":  # FP64 fast path
        assert np.abs(mine - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["trace", "info"])
def test_quad_exact_mode_bit_identical(g_small, models, small_grid, kind):
    f = F.Field.build(g_small["points"], small_grid, models["quad"], kind, exact=True)
    assert np.array_equal(reference_order(f), g_small[f"factors_quad_{kind}"])
    f7 = F.Field.build(g_small["points"], small_grid, models["quad"], "info", sigma=0.7, exact=True)
    assert np.array_equal(reference_order(f7), g_small["factors_quad_info_sigma07"])


def test_config1_sampled_rows(g_cfg1, models):
    """Config-1 landmark set (2 000) on 24 sampled voxels, explicit-centre mode."""
    dev = torch.device("cuda")
    pts = torch.tensor(g_cfg1["points"], device=dev)
    cs = torch.tensor(g_cfg1["centers"], device=dev)
    for mname in ("quad", "gp70"):
        for kind in ("trace", "info"):
            m = models[mname]
            s64, _ = FD.build_rows(pts, m, kind == "trace", 1.0, dev, centers=cs, exact=(mname == "quad"))
            fld = FD.Field(F.GridConfig(np.zeros(3), 1.0, np.array([24, 1, 1])), m, kind, 1.0, s64, None,
                           np.stack([np.arange(24), np.zeros(24), np.zeros(24)], 1), dense=False)
            mine, ref = fld.factors, g_cfg1[f"{mname}_{kind}"]
            if mname == "quad":
                assert np.array_equal(mine, ref)
            else:
                err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
                assert err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL)


@pytest.mark.parametrize("mname", ["quad", "gp70"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_config1_full_grid_vs_oracle(oracle, models, mname, kind, gp_info_kernel):
    """Every voxel of BASELINE config 1 (21x21x7 grid, 2 000 uniform landmarks)."""
    from paper_2008_03324_b200 import scenes

    w = scenes.config1(0)
    grid = F.GridConfig(*w.grid)
    f = F.Field.build(w.points, grid, models[mname], kind)
    mine = reference_order(f)
    ref = oracle_field(oracle, models[mname], grid.centers(), w.points, kind)
    err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
    assert err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL)


@pytest.mark.parametrize("mname", ["quad", "gp70"])
def test_config2_sampled_voxels(oracle, models, mname, gp_info_kernel):
    """BASELINE config 2 (20 000 float32 room landmarks) on random + boundary voxels."""
    from paper_2008_03324_b200 import scenes

    w = scenes.config2(0)
    grid = F.GridConfig(*w.grid)
    rng = np.random.default_rng(9)
    idx3 = grid.index3_of(rng.choice(grid.voxel_count, 40, replace=False))
    corners = np.array([[i, j, k] for i in (0, 80) for j in (0, 80) for k in (0, 20)])
    idx3 = np.vstack([idx3, corners])
    cen = grid.center_of(idx3)
    dev = torch.device("cuda")
    pts = torch.tensor(w.points, device=dev)
    for kind in ("trace", "info"):
        s64, _ = FD.build_rows(pts, models[mname], kind == "trace", 1.0, dev, centers=torch.tensor(cen, device=dev))
        fld = FD.Field(grid, models[mname], kind, 1.0, s64, None, idx3.astype(np.int32), dense=False)
        ref = oracle_field(oracle, models[mname], cen, w.points, kind)
        err = trace_rel_l2(fld.factors, ref) if kind == "trace" else info_rel_fro(fld.factors, ref)
        assert err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL)


def test_linearity_and_slab_determinism(models, small_grid, g_small):
    """field(S1 u S2) == field(S1) + field(S2) and the z-slab pieces of a
    sharded build are bit-identical to the single build."""
    from paper_2008_03324_b200.parallel import slab_range

    dev = torch.device("cuda")
    pts = g_small["points"]
    for mname, tol in (("quad", 1e-12), ("gp30", 1e-5)):  # GP: FP32/TF32 per-pair math, FP32 partial sums
        m = models[mname]
        full = F.Field.build(pts, small_grid, m, "info")
        a = F.Field.build(pts[:150], small_grid, m, "info")
        b = F.Field.build(pts[150:], small_grid, m, "info")
        s = a.storage["f64"] + b.storage["f64"]
        ref = full.storage["f64"]
        assert (torch.abs(s - ref).max() / torch.abs(ref).max()).item() < tol
        P = torch.tensor(pts, device=dev)
        V = small_grid.voxel_count
        for world in (2, 3, 8):
            parts = [FD.build_rows(P, m, False, 1.0, dev, grid=small_grid, v_begin=b0, v_end=b1)[0]
                     for b0, b1 in (slab_range(V, world, r) for r in range(world))]
            assert torch.equal(torch.cat(parts), ref)


def test_empty_and_degenerate(models, oracle):
    grid = F.GridConfig(np.array([0.0, 0.0, 0.0]), 1.0, np.array([3, 2, 2]))
    f = F.Field.build(np.zeros((0, 3)), grid, models["quad"], "info")
    assert f.rows == 0 and (f.slots == -1).all()
    fims, ok = f.query_fim_batch(np.array([[1.2, 1.1, 1.0]]), np.eye(3)[None], "trilinear")
    assert ok[0] and np.all(fims == 0)
    # a landmark exactly at a voxel centre is skipped, like kernels.py:444
    c = grid.centers()
    pts = np.vstack([c[3], [5.0, 4.0, 3.0], c[7] + 1e-3])
    for mname in ("quad", "gp30"):
        for kind in ("trace", "info"):
            ff = F.Field.build(pts, grid, models[mname], kind, exact=(mname == "quad"))
            ref = oracle_field(oracle, models[mname], c, pts, kind)
            mine = reference_order(ff)
            if mname == "quad":
                assert np.array_equal(mine, ref)
            else:
                err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
                assert np.isfinite(mine).all() and err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL)


def test_matchability_mask(models, oracle, g_small, small_grid):
    """Range-gated matchability (field.py:152-158): mask applied in-kernel, occupied rows only."""
    mt = F.Matchability(d_near=0.3, d_far=1.6)
    pts = g_small["points"]
    for mname in ("quad", "gp30"):
        f = F.Field.build(pts, small_grid, models[mname], "info", matchability=mt)
        mask = mt.mask(small_grid.centers(), pts)
        occ = mask.any(axis=1)
        ref = oracle_field(oracle, models[mname], small_grid.centers()[occ], pts, "info", mask=mask[occ])
        assert f.rows == occ.sum()
        assert np.array_equal(small_grid.linear_index(f.occupied_index3), np.nonzero(occ)[0])
        assert info_rel_fro(f.factors, ref).max() <= INFO_TOL


def test_incremental_add_remove(models, small_grid, g_small):
    """add/remove == rebuild; quad is FP64 throughout, GP's FP32 partial sums
    group landmarks differently in the two builds, so agreement is at FP32-partial level."""
    pts = g_small["points"]
    for mname, tol in (("quad", 1e-12), ("gp30", 1e-5)):
        full = F.Field.build(pts, small_grid, models[mname], "info")
        inc = F.Field.build(pts[:200], small_grid, models[mname], "info")
        inc.add_landmarks(pts[200:])
        ref = full.storage["f64"]
        assert (torch.abs(inc.storage["f64"] - ref).max() / torch.abs(ref).max()).item() < tol
        inc.remove_landmarks(pts[200:])
        base = F.Field.build(pts[:200], small_grid, models[mname], "info").storage["f64"]
        assert (torch.abs(inc.storage["f64"] - base).max() / torch.abs(base).max()).item() < tol


def test_serialize_roundtrip(models, small_grid, g_small, tmp_path):
    for mname in ("quad", "gp30"):
        f = F.Field.build(g_small["points"], small_grid, models[mname], "info")
        p = tmp_path / f"{mname}.fif"
        f.serialize(p)
        g = F.Field.deserialize(p)
        assert np.array_equal(g.factors, f.factors[np.argsort(small_grid.linear_index(f.occupied_index3))])
        pos = g_small["positions"][:50]
        rots = g_small["rotations"][:50]
        a, oka = f.query_fim_batch(pos, rots, "trilinear")
        b, okb = g.query_fim_batch(pos, rots, "trilinear")
        assert np.array_equal(oka, okb)
        # quad: FP64 rows round-trip exactly; GP: S = K F is re-rounded to the FP32 query copy
        tol = 1e-12 if mname == "quad" else 1e-6
        assert np.abs(a - b).max() <= tol * np.abs(a).max()
    # a field with no rows (empty landmark set, or matchability rejecting every voxel) is a
    # valid FIF1 file, as the reference writes it: it round-trips
    for mname in ("quad", "gp30"):
        for kind in ("trace", "info"):
            e = F.Field.build(np.zeros((0, 3)), small_grid, models[mname], kind)
            pe = tmp_path / f"empty_{mname}_{kind}.fif"
            e.serialize(pe)
            ge = F.Field.deserialize(pe)
            assert ge.rows == 0 and (ge.slots == -1).all()
            fims, ok = ge.query_fim_batch(g_small["positions"][:4], g_small["rotations"][:4], "trilinear") \
                if kind == "info" else (None, None)
            if kind == "info":
                assert np.all(fims == 0)
    with pytest.raises(F.BadMagic):
        bad = tmp_path / "bad.fif"
        bad.write_bytes(b"XXXX" + b"\0" * 64)
        F.Field.deserialize(bad)


@pytest.mark.parametrize("kind", ["trace", "info"])
def test_gp150_build(oracle, kind, gp_info_kernel):
    """N_s = 150 (the largest GP size of the paper's Table I; two warps per voxel on the
    tensor path) on a small scene vs the oracle."""
    m = F.build_gp_model(150)
    rng = np.random.default_rng(12)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(300, 3))
    grid = F.GridConfig(np.array([-1.0, -1.0, 0.25]), 0.5, np.array([4, 3, 3]))
    f = F.Field.build(pts, grid, m, kind)
    ref = oracle_field(oracle, m, grid.centers(), pts, kind)
    mine = reference_order(f)
    err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
    assert err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL)


def test_fif1_interop_with_reference_files(tmp_path, g_models):
    """FIF1 files written by the reference's Field.serialize (tests/golden/fif1) load here,
    and an EXACT-mode quad build serialises byte-for-byte like the reference's."""
    import os

    from tests._helpers import models_from_golden

    d = os.path.join(os.path.dirname(__file__), "golden", "fif1")
    inp = np.load(os.path.join(d, "inputs.npz"))
    cfg = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([4, 3, 3]))
    m = models_from_golden(g_models)
    # quad info: bit-exact build -> identical bytes
    ours = F.Field.build(inp["points"], cfg, m["quad"], "info", exact=True)
    p = tmp_path / "q.fif"
    ours.serialize(p)
    assert p.read_bytes() == open(os.path.join(d, "quad_info.fif"), "rb").read()
    # the reference's files deserialise to the same rows the build produces
    for name, model, kind in (("quad_info", m["quad"], "info"), ("gp30_trace", m["gp30"], "trace")):
        g = F.Field.deserialize(os.path.join(d, name + ".fif"))
        assert g.factor_kind == kind and g.rows == cfg.voxel_count
        ref = F.Field.build(inp["points"], cfg, model, kind, exact=isinstance(model, F.QuadraticVisibility))
        order = np.argsort(cfg.linear_index(ref.occupied_index3))
        a, b = g.factors, ref.factors[order]
        assert np.abs(a - b).max() <= (0.0 if kind == "info" else 1e-5 * np.abs(b).max())
    # masked GP info (sparse rows in the reference's order) loads and queries
    g = F.Field.deserialize(os.path.join(d, "gp30_info_masked.fif"))
    assert g.factor_kind == "info" and 0 < g.rows <= cfg.voxel_count
    q = g.query_batch(cfg.centers()[:5], axes=np.tile([0.0, 0.0, 1.0], (5, 1)), outputs=("trace",), mode="nearest")
    assert torch.isfinite(q["trace"]).all()


@pytest.mark.parametrize("k_s", [60.0, 200.0])
def test_sharp_sigmoids_stay_finite(oracle, g_small, models, small_grid, k_s, gp_info_kernel):
    """Sharp visibility sigmoids: exponent arguments |x| = k_s |u.z - cos a| log2(e) reach
    ~500, far past FP32's 2^x range and the trace kernel's paired-reciprocal clamp
    (x <= 63); the builds stay finite and within tolerance of the oracle."""
    m0 = models["gp30"]
    m = F.GpVisibility(m0.samples, m0.params, m0.alpha, k_s, m0.kinv)
    pts = g_small["points"]
    cen = small_grid.centers()
    for kind in ("trace", "info"):
        mine = reference_order(F.Field.build(pts, small_grid, m, kind))
        assert np.isfinite(mine).all()
        ref = oracle_field(oracle, m, cen, pts, kind)
        err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
        assert err.max() <= (TRACE_TOL if kind == "trace" else INFO_TOL), (kind, err.max())


@pytest.mark.parametrize("mname,kind", [("gp30", "info"), ("gp70", "info"), ("quad", "info"), ("gp70", "trace")])
def test_build_host_factors_pipelined(models, mname, kind):
    """Field.build(host_factors=True): z-slab chunks whose export + D2H overlap the next
    chunk's build return the same host factors (bit for bit) and device rows as the
    one-launch build followed by export_reference; export_reference_to likewise."""
    from paper_2008_03324_b200 import scenes as SC

    w = SC.config1(0)
    grid = F.GridConfig(*w.grid)
    model = models[mname] if mname in models else F.build_gp_model(int(mname[2:]))
    ref = F.Field.build(w.points, grid, model, kind)
    want = ref.export_reference().cpu().numpy()
    got = F.Field.build(w.points, grid, model, kind, host_factors=True)
    assert got.factors.shape == want.shape and np.array_equal(got.factors, want)
    assert torch.equal(got.storage["f64"], ref.storage["f64"])
    host = torch.empty(want.shape, dtype=torch.float64).pin_memory()
    again = F.Field.build(w.points, grid, model, kind, host_factors=True, host_out=host)
    assert np.array_equal(host.numpy(), want) and again.factors.ctypes.data == host.numpy().ctypes.data
    assert np.array_equal(ref.export_reference_to(chunk_rows=777), want)
    with pytest.raises(ValueError):
        F.Field.build(w.points, grid, model, kind, host_factors=True, host_out=torch.empty((3, 3), dtype=torch.float64))


@pytest.mark.parametrize("ns", [4, 5, 9, 16, 20, 21, 28, 29])
def test_small_sample_counts_trace_and_info(oracle, ns):
    """GP fields with few samples (kernels.py:471-524 takes any N_s): the trace kernel packs
    more voxels per CTA the fewer samples there are (N_s <= 20 once asked for more shared
    memory than its opt-in: found by tools/soak_masked.py), the info build runs the small
    tcgen05 / mma.sync instantiations; queries on both."""
    rng = np.random.default_rng(100 + ns)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(300, 3))
    grid = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([4, 3, 2]))
    m = F.build_gp_model(ns, length_scale=0.5)
    for kind, tol in (("trace", 1e-5), ("info", 1e-4)):
        f = F.Field.build(pts, grid, m, kind)
        ref = oracle_field(oracle, m, grid.centers(), pts, kind)
        mine = reference_order(f)
        err = trace_rel_l2(mine, ref) if kind == "trace" else info_rel_fro(mine, ref)
        assert err.max() <= tol, (kind, ns, err.max())
        fm = F.Field.build(pts, grid, m, kind, matchability=F.Matchability(d_far=2.5))
        refm = oracle_field(oracle, m, grid.centers(), pts, kind,
                            mask=np.asarray(F.Matchability(d_far=2.5).mask(grid.centers(), pts), dtype=np.uint8))
        idx = grid.linear_index(fm.occupied_index3)
        errm = (trace_rel_l2 if kind == "trace" else info_rel_fro)(fm.factors, refm[idx])
        assert errm.max() <= tol, (kind, ns, "masked", errm.max())

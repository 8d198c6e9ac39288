"""Matchability gates (field.py:101-180) against the reference's own masks and
masked builds (tests/golden/make_golden_match.py)."""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from tests._helpers import info_rel_fro, models_from_golden, trace_rel_l2

CASES = {
    "range": lambda g: F.Matchability(d_near=float(g["d_near"]), d_far=float(g["d_far"])),
    "near": lambda g: F.Matchability(d_near=float(g["d_near"])),
    "cone": lambda g: F.Matchability(view_cone_beta=1.1),
    "range_cone": lambda g: F.Matchability(d_near=0.4, d_far=2.2, view_cone_beta=0.9),
    "sparse": lambda g: F.Matchability(d_near=0.3, d_far=0.75, view_cone_beta=0.8),
}
GRID = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([6, 5, 4]))


@pytest.mark.parametrize("name", ["range", "near", "cone", "range_cone"])
def test_host_mask_matches_reference(g_match, name):
    mt = CASES[name](g_match)
    mine = mt.mask(g_match["centers"], g_match["points"], g_match["view_dirs"])
    assert np.array_equal(mine, g_match[f"mask_{name}"])


def test_limits_are_inclusive(g_match):
    m = g_match["mask_range"]
    assert m[7, 11] == 1 and m[23, 42] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["range", "near", "cone", "range_cone"])
def test_device_mask_bit_exact(g_match, name):
    dev = torch.device("cuda")
    mt = CASES[name](g_match)
    m = mt.device_mask(torch.tensor(g_match["centers"], device=dev), torch.tensor(g_match["points"], device=dev),
                       g_match["view_dirs"])
    assert np.array_equal(m.cpu().numpy(), g_match[f"mask_{name}"])


@pytest.mark.gpu
def test_device_mask_with_host_predicate(g_match):
    """Host-only gates (Python predicate) AND the GPU gates, as the reference composes them."""
    dev = torch.device("cuda")
    pred = lambda c, p: p[2] > 0.5  # noqa: E731
    mt = F.Matchability(d_near=0.4, d_far=2.2, predicate=pred)
    m = mt.device_mask(torch.tensor(g_match["centers"], device=dev), torch.tensor(g_match["points"], device=dev))
    ref = mt.mask(g_match["centers"], g_match["points"])
    assert np.array_equal(m.cpu().numpy(), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("mname", ["quad", "gp30"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_masked_build_vs_reference(g_match, g_models, mname, kind):
    """fifield.build(scene, ..., matchability=range+cone) reproduced: occupied rows in
    the reference's order and factors within the BASELINE tolerances."""
    models = models_from_golden(g_models)
    scene = F.Scene(g_match["points"], g_match["view_dirs"])
    f = F.build(scene, GRID, models[mname], kind, matchability=CASES["sparse"](g_match))
    assert np.array_equal(f.occupied_index3, g_match[f"occ3_{mname}_{kind}"])
    ref = g_match[f"factors_{mname}_{kind}"]
    if mname == "quad":
        err = np.abs(f.factors - ref).max() / np.abs(ref).max()
        assert err <= 1e-12
    else:
        err = trace_rel_l2(f.factors, ref) if kind == "trace" else info_rel_fro(f.factors, ref)
        assert err.max() <= (1e-5 if kind == "trace" else 1e-4)


@pytest.mark.gpu
def test_masked_incremental(g_match, g_models):
    models = models_from_golden(g_models)
    mt = CASES["sparse"](g_match)
    pts, vd = g_match["points"], g_match["view_dirs"]
    full = F.build(F.Scene(pts, vd), GRID, models["quad"], "info", matchability=mt)
    inc = F.build(F.Scene(pts[:150], vd[:150]), GRID, models["quad"], "info", matchability=mt)
    inc.add_landmarks(F.Scene(pts[150:], vd[150:]))
    order = np.argsort(GRID.linear_index(inc.occupied_index3))
    assert np.array_equal(GRID.linear_index(inc.occupied_index3)[order], GRID.linear_index(full.occupied_index3))
    a, b = inc.factors[order], full.factors
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


# ── ObstacleWorld occlusion (world.segment_blocked, world.py:96-140) ──
class _Sphere:
    def __init__(self, c, r):
        self.center, self.radius = np.asarray(c), float(r)


class _Box:
    def __init__(self, lo, hi):
        self.lo, self.hi = np.asarray(lo), np.asarray(hi)


class _World:
    """Duck-typed stand-in for fifield.world.ObstacleWorld (spheres / boxes lists)."""

    def __init__(self, spheres, boxes):
        self.spheres = [_Sphere(s[:3], s[3]) for s in spheres]
        self.boxes = [_Box(b[:3], b[3:]) for b in boxes]


def _occ_cases(g):
    w = _World(g["spheres"], g["boxes"])
    return {"occ": F.Matchability(occluders=w), "occ_range": F.Matchability(d_near=0.3, d_far=2.4, occluders=w),
            "occ_all": F.Matchability(d_near=0.2, d_far=3.0, view_cone_beta=1.2, occluders=w)}


@pytest.fixture(scope="module")
def g_occ():
    import os

    return np.load(os.path.join(os.path.dirname(__file__), "golden", "match_occ.npz"))


@pytest.mark.parametrize("name", ["occ", "occ_range", "occ_all"])
def test_host_occlusion_mask_matches_reference(g_occ, name):
    mt = _occ_cases(g_occ)[name]
    assert np.array_equal(mt.mask(g_occ["centers"], g_occ["points"], g_occ["view_dirs"]), g_occ[f"mask_{name}"])
    assert np.array_equal(_occ_cases(g_occ)["occ"].mask(g_occ["centers"], g_occ["points"][400:401]),
                          g_occ["mask_single"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["occ", "occ_range", "occ_all"])
def test_device_occlusion_mask_bit_exact(g_occ, name):
    dev = torch.device("cuda")
    mt = _occ_cases(g_occ)[name]
    c, p = torch.tensor(g_occ["centers"], device=dev), torch.tensor(g_occ["points"], device=dev)
    m = mt.device_mask(c, p, g_occ["view_dirs"])
    assert np.array_equal(m.cpu().numpy(), g_occ[f"mask_{name}"])
    any_ = mt.device_any(c, p, g_occ["view_dirs"]).cpu().numpy()
    assert np.array_equal(any_, g_occ[f"mask_{name}"].any(axis=1))
    single = _occ_cases(g_occ)["occ"].device_mask(c, p[400:401].contiguous())
    assert np.array_equal(single.cpu().numpy(), g_occ["mask_single"])


@pytest.mark.gpu
@pytest.mark.parametrize("mname", ["quad", "gp30"])
@pytest.mark.parametrize("kind", ["trace", "info"])
def test_fused_occlusion_build_vs_reference(g_occ, g_models, mname, kind):
    """Range + view cone + occlusion evaluated inside the build kernels (fif_build_matched):
    the reference's occupied rows and factors, with no (V, N) mask allocated."""
    models = models_from_golden(g_models)
    scene = F.Scene(g_occ["points"], g_occ["view_dirs"])
    f = F.build(scene, GRID, models[mname], kind, matchability=_occ_cases(g_occ)["occ_all"])
    assert np.array_equal(f.occupied_index3, g_occ[f"occ3_{mname}_{kind}"])
    ref = g_occ[f"factors_{mname}_{kind}"]
    if mname == "quad":
        assert np.abs(f.factors - ref).max() <= 1e-12 * np.abs(ref).max()
    else:
        err = trace_rel_l2(f.factors, ref) if kind == "trace" else info_rel_fro(f.factors, ref)
        assert err.max() <= (1e-5 if kind == "trace" else 1e-4)


@pytest.mark.gpu
def test_fused_gates_equal_explicit_mask_build(g_match, g_models):
    """The fused-gate build is bit-identical to the explicit-mask build of the same pairs
    (same kernels, same per-pair decisions), for every GP-info kernel variant."""
    from paper_2008_03324_b200 import field as FD

    models = models_from_golden(g_models)
    dev = torch.device("cuda")
    mt = CASES["range_cone"](g_match)
    pts = torch.tensor(g_match["points"], device=dev)
    cen = torch.tensor(g_match["centers"], device=dev)
    mask = mt.device_mask(cen, pts, g_match["view_dirs"])
    for mname in ("quad", "gp30"):
        for kind in (True, False):
            for kern in (("t5", "h16", "tf32", "simt") if mname == "gp30" and not kind else ("t5",)):
                old = FD.GP_INFO_KERNEL
                FD.GP_INFO_KERNEL = kern
                try:
                    a, _ = FD.build_rows(pts, models[mname], kind, 1.0, dev, centers=cen, mask=mask)
                    b, _ = FD.build_matched_rows(pts, models[mname], kind, 1.0, dev, cen, mt, g_match["view_dirs"])
                finally:
                    FD.GP_INFO_KERNEL = old
                assert torch.equal(a, b), (mname, kind, kern)

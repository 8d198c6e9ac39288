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

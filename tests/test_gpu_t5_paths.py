"""Edge paths of the tcgen05 GP-info build (k_gp_info_t5): the fallback to the mma.sync
kernel when the paired sigmoid reciprocal is not safe (x = (ax zs).u + bx above 60), the
masked build with too many landmarks for the shared-memory gate bits (gates evaluated in
both passes), odd N_s (a padded sample column), and a landmark almost on a voxel centre
(the pre-pass bound sets the FP16 scale from it)."""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD

from ._helpers import info_rel_fro, oracle_field

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda")


def _grid():
    return F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([4, 4, 2]))


def _check(oracle, model, pts, grid, kern="t5"):
    old = FD.GP_INFO_KERNEL
    FD.GP_INFO_KERNEL = kern
    try:
        f = F.Field.build(pts, grid, model, "info")
    finally:
        FD.GP_INFO_KERNEL = old
    mine = f.factors[np.argsort(grid.linear_index(f.occupied_index3))]
    ref = oracle_field(oracle, model, grid.centers(), pts, "info")
    return info_rel_fro(mine, ref).max()


def test_sharp_sigmoid_falls_back_and_matches(oracle):
    """k_s = 40: bx + |ax| ~ 98 > 60, so the host routes the build to k_gp_info_h16."""
    rng = np.random.default_rng(11)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(500, 3))
    m = F.build_gp_model(30, k_s=40.0)
    assert _check(oracle, m, pts, _grid()) <= 1e-4


@pytest.mark.parametrize("ns", [21, 45, 79])
def test_odd_sample_counts(oracle, ns):
    rng = np.random.default_rng(ns)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(700, 3))
    assert _check(oracle, F.build_gp_model(ns), pts, _grid()) <= 1e-4


def test_landmark_near_a_voxel_centre(oracle):
    grid = _grid()
    rng = np.random.default_rng(5)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(400, 3))
    c = grid.centers()
    pts[0] = c[5] + np.array([3e-6, -2e-6, 1e-6])  # w ~ 1e11: sets the voxel's FP16 scale
    pts[1] = c[9]                                     # exactly on a centre: skipped (n^2 == 0)
    assert _check(oracle, F.build_gp_model(70), pts, grid) <= 1e-4


@pytest.mark.parametrize("ns, n", [(30, 100_000), (70, 20_000), (70, 100_000)])
def test_masked_build_gate_bits(oracle, ns, n):
    """Masked builds, 4 voxels (slots 0-2 of one CTA and slot 0 of the next).  N_s = 30 at
    1e5 and N_s = 70 at 2e4 landmarks keep the pre-pass's gate answers as bits in shared
    memory ([voxel][n_pad / 32] words; n_pad not a multiple of the pre-pass stride, the
    case where a voxel's trailing words once spilled into the next voxel's); N_s = 70 at
    1e5 has no room for them and evaluates the gate in the pre-pass and again per tile."""
    rng = np.random.default_rng(3)
    pts = rng.uniform([-6, -6, -1], [6, 6, 3], size=(n, 3))
    grid = F.GridConfig(np.array([-0.5, -0.5, 0.5]), 0.5, np.array([2, 2, 1]))
    cen = grid.centers()
    m = F.build_gp_model(ns)
    mt = F.Matchability(d_near=0.3, d_far=4.0)
    s64, _ = FD.build_matched_rows(torch.tensor(pts, device=DEV), m, False, 1.0, DEV, torch.tensor(cen, device=DEV), mt)
    mask = mt.mask(cen, pts)
    ref = oracle_field(oracle, m, cen, pts, "info", mask=np.asarray(mask, dtype=np.uint8))
    fld = FD.Field(grid, m, "info", 1.0, s64, None, grid.index3_of(np.arange(cen.shape[0])).astype(np.int32), dense=False)
    assert info_rel_fro(fld.factors, ref).max() <= 1e-4

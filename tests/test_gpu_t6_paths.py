"""k_gp_info_t6 (FIF_BUILD_T6): the GP-info build with the sigmoid exponent arguments on the
tensor cores (X = A_x B_x^T, FP16 u hi + lo against z hi + mid + lo) and the merged hi / lo S
accumulators.  Same tolerances as the default kernel: max entry error <= 1e-4 of the voxel's
Frobenius norm against the FP64 oracle (kernels.py:471-524); every N_s group count the kernel
is instantiated for (with and without a skipped padding pair), the fallback outside its
range, a landmark almost on a voxel centre, z-slab bit-determinism and config-2 voxels."""
import numpy as np
import pytest
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC

from ._helpers import info_rel_fro, oracle_field

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda")


@pytest.fixture(autouse=True)
def _t6():
    old = FD.GP_INFO_KERNEL
    FD.GP_INFO_KERNEL = "t6"
    yield
    FD.GP_INFO_KERNEL = old


def _grid():
    return F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([4, 4, 2]))


def _err(oracle, model, pts, grid):
    f = F.Field.build(pts, grid, model, "info")
    mine = f.factors[np.argsort(grid.linear_index(f.occupied_index3))]
    ref = oracle_field(oracle, model, grid.centers(), pts, "info")
    return info_rel_fro(mine, ref).max()


@pytest.mark.parametrize("ns", [9, 16, 22, 24, 30, 40, 45, 48, 54, 64, 70, 71, 72])
def test_sample_counts(oracle, ns):
    """N_s = 9 .. 72 (NG = 2 .. 9 sample groups; N_s <= 8 NG - 2 skips one padding pair)."""
    rng = np.random.default_rng(ns)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(700, 3))
    assert _err(oracle, F.build_gp_model(ns), pts, _grid()) <= 1e-4


@pytest.mark.parametrize("ns, k_s", [(8, 15.0), (79, 15.0), (30, 40.0)])
def test_outside_the_kernels_range_falls_back(oracle, ns, k_s):
    """N_s <= 8, N_s > 72 and sharp sigmoids run the default kernels under the same flag."""
    rng = np.random.default_rng(7)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(500, 3))
    assert _err(oracle, F.build_gp_model(ns, k_s=k_s), pts, _grid()) <= 1e-4


def test_landmark_near_a_voxel_centre_and_odd_tiles(oracle):
    grid = _grid()
    rng = np.random.default_rng(5)
    pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(1100, 3))  # 18 tiles: a partial last span
    c = grid.centers()
    pts[0] = c[5] + np.array([3e-6, -2e-6, 1e-6])  # w ~ 1e11: sets the voxel's FP16 scale
    pts[1] = c[9]                                     # exactly on a centre: skipped (n^2 == 0)
    assert _err(oracle, F.build_gp_model(70), pts, grid) <= 1e-4


def test_slab_and_centre_list_determinism():
    """A voxel's rows do not depend on the CTA slot, slab or centre list it is built in."""
    from paper_2008_03324_b200.parallel import slab_range

    rng = np.random.default_rng(2)
    pts = torch.tensor(rng.uniform([-3, -3, 0], [3, 3, 2], size=(1500, 3)), device=DEV)
    grid = F.GridConfig(np.array([-1.0, -1.0, 0.0]), 0.4, np.array([5, 4, 3]))
    m = F.build_gp_model(70)
    V = grid.voxel_count
    ref = FD.build_rows(pts, m, False, 1.0, DEV, grid=grid)[0]
    for world in (2, 3, 7):
        parts = [FD.build_rows(pts, m, False, 1.0, DEV, grid=grid, v_begin=b0, v_end=b1)[0]
                 for b0, b1 in (slab_range(V, world, r) for r in range(world))]
        assert torch.equal(torch.cat(parts), ref)


def test_config2_sampled_voxels_and_t5_agreement(oracle):
    w = SC.config2(10)
    grid = F.GridConfig(*w.grid)
    m = F.build_gp_model(70)
    rng = np.random.default_rng(1)
    sample = np.sort(rng.choice(grid.voxel_count, 200, replace=False))
    cen = grid.centers()[sample]
    pts = torch.tensor(w.points, device=DEV)
    cd = torch.tensor(cen, device=DEV)
    r6 = FD.build_rows(pts, m, False, 1.0, DEV, centers=cd)[0]
    FD.GP_INFO_KERNEL = "t5"
    r5 = FD.build_rows(pts, m, False, 1.0, DEV, centers=cd)[0]
    assert (torch.abs(r6 - r5).max() / torch.abs(r5).max()).item() < 5e-6
    # pre-kinv sums against the oracle's (kinv = identity), max entry / voxel Frobenius
    ref = oracle.build_gp_factors(cen, np.asarray(w.points, dtype=np.float64), 1.0, m.samples, np.eye(70), m.k_s,
                                  np.cos(m.alpha), False)
    iu = np.triu_indices(6)
    refp = ref.reshape(len(sample), 70, 6, 6)[:, :, iu[0], iu[1]].reshape(len(sample), -1)
    err = np.abs(r6.cpu().numpy() - refp).max(1) / np.linalg.norm(refp, axis=1)
    assert err.max() <= 1e-5

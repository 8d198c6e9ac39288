"""CPU tests of the host side: model parameters vs the reference fixtures, geometry,
grid bookkeeping, workload generators, the C-ABI library's exports."""
import os
import re

import numpy as np
import pytest

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import _lib, scenes
from paper_2008_03324_b200.field import GridConfig, _from_reference_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gp_models_bit_identical_to_reference(g_models):
    """Host restatement of build_gp_model / gp_build / train_lengthscale (visibility.py:249-374)
    reproduces the reference's length scale and kinv exactly."""
    for ns in (30, 70):
        m = F.build_gp_model(ns)
        par = g_models[f"gp{ns}_par"]
        assert m.params.length_scale == par[3]
        assert np.array_equal(m.kinv, g_models[f"gp{ns}_kinv"])
        assert np.array_equal(m.samples, g_models[f"gp{ns}_zs"])
    fixed = F.gp_build(F.sample_directions(30), F.SeKernelParams(1.0, 0.5))
    assert np.array_equal(fixed.kinv, g_models["gp30_l05_kinv"])
    l = F.train_lengthscale(50, F.sample_directions(20), search_grid=np.geomspace(0.1, 1.5, 8), seed=2)
    assert l == g_models["train_l_small"][0]


def test_quad_coefficients(g_models):
    for a, va, k2, k1, k0 in g_models["quad_coeffs_grid"]:
        assert F.quad_coefficients(a, va) == (k2, k1, k0)
    with pytest.raises(F.SingularFov):
        F.quad_coefficients(1e-12, 0.5)


def test_model_kats():
    """test_visibility.py:28-73, 112-147 restated against this package."""
    k2, k1, k0 = F.quad_coefficients(np.pi / 4, 0.5)
    assert k2 == pytest.approx(np.sqrt(2) / 2, abs=1e-12) and k1 == 0.5
    m = F.build_quad_model()
    rng = np.random.default_rng(0)
    t = rng.standard_normal(3)
    p = t + rng.standard_normal(3) * 3
    R = F.random_rotation(rng)
    u = (p - t) / np.linalg.norm(p - t)
    assert m.value(R, t, p) == pytest.approx(m.value_cos(float(R[:, 2] @ u)), abs=1e-12)
    zs = F.sample_directions(30)
    g = F.gp_build(zs, F.SeKernelParams(1.0, 0.5))
    gram = np.array([[F.se_kernel(a, b, F.SeKernelParams(1.0, 0.5)) for b in zs] for a in zs])
    np.testing.assert_allclose(g.kinv @ gram, np.eye(30), atol=1e-5)
    with pytest.raises(F.SingularGram):
        F.gp_build(np.tile([[0.0, 0.0, 1.0]], (8, 1)), F.SeKernelParams(1.0, 0.5, jitter=0.0))
    with pytest.raises(ValueError):
        F.gp_build(np.eye(3), F.SeKernelParams())
    with pytest.raises(F.TooFewSamples):
        F.sample_directions(3)


def test_landmark_fim_and_jacobian_kats(g_kats):
    for i in range(g_kats["t"].shape[0]):
        np.testing.assert_allclose(F.landmark_fim(g_kats["t"][i], g_kats["p"][i], g_kats["sigma"][i]),
                                   g_kats["fim"][i], rtol=1e-12, atol=1e-14)
        pose = F.Pose(g_kats["rot"][i], g_kats["t"][i])
        np.testing.assert_allclose(F.bearing_jacobian(pose, g_kats["p"][i]), g_kats["jac"][i], rtol=1e-12,
                                   atol=1e-14)
    with pytest.raises(F.DegeneratePoint):
        F.landmark_fim(np.ones(3), np.ones(3))
    m = F.landmark_fim(np.zeros(3), np.array([2.0, 1.0, 3.0]))
    assert np.linalg.matrix_rank(m, tol=1e-9) == 2


def test_geometry(g_kats):
    assert np.array_equal(F.sample_directions(70), g_kats["fib70"])
    assert np.array_equal(F.sample_directions(7), g_kats["fib7"])
    rng = np.random.default_rng(3)
    R = F.random_rotation(rng)
    assert np.allclose(R.T @ R, np.eye(3)) and np.linalg.det(R) > 0
    assert F.wrap_angle(np.pi) == pytest.approx(np.pi)
    assert F.wrap_angle(-np.pi) == pytest.approx(np.pi)
    Rb = scenes.uniform_rotations(np.random.default_rng(3), 5)
    rng = np.random.default_rng(3)
    q = rng.standard_normal((5, 4))
    assert np.allclose(Rb, scenes.quat_to_rot(q))


def test_grid_bookkeeping(g_small):
    g = GridConfig(g_small["origin"], g_small["voxel_size"][0], g_small["dims"])
    assert np.array_equal(g.centers(), g_small["centers"])
    lin = np.arange(g.voxel_count)
    i3 = g.index3_of(lin)
    assert np.array_equal(g.linear_index(i3), lin)
    j = g.internal_index(i3)
    assert np.array_equal(np.sort(j), lin)
    assert np.array_equal(g.index3_of_internal(j), i3)
    with pytest.raises(F.EmptyGrid):
        GridConfig(np.zeros(3), 1.0, np.array([0, 1, 1]))
    with pytest.raises(ValueError):
        GridConfig(np.zeros(3), 0.0, np.array([1, 1, 1]))


def test_reference_row_conversion(g_small, g_models):
    """Reference-layout rows -> packed device layout keeps exactly the upper triangle (quad)
    and maps GP rows to S = K F."""
    from tests._helpers import models_from_golden

    ms = models_from_golden(g_models)
    F36 = g_small["factors_quad_info"]
    packed = _from_reference_rows(F36, ms["quad"], "info")
    blocks = F36.reshape(-1, 10, 6, 6)
    assert np.array_equal(blocks, np.transpose(blocks, (0, 1, 3, 2)))
    iu = np.triu_indices(6)
    assert np.array_equal(packed.reshape(-1, 10, 21), blocks[:, :, iu[0], iu[1]])
    G = g_small["factors_gp30_trace"]
    S = _from_reference_rows(G, ms["gp30"], "trace")
    np.testing.assert_allclose(S @ ms["gp30"].kinv.T, G, rtol=1e-8, atol=1e-9 * np.abs(G).max())


def test_workload_generators():
    w1 = scenes.config1(10)
    assert w1.points.shape == (2000, 3) and w1.positions.shape == (10, 3)
    ref = np.random.default_rng(0).uniform([-5, -5, 0], [5, 5, 3], size=(2000, 3))
    assert np.array_equal(w1.points, ref)
    w2 = scenes.config2(5)
    assert w2.points.shape == (20000, 3)
    assert np.array_equal(w2.points, w2.points.astype(np.float32).astype(np.float64))
    assert (np.abs(w2.points[:, :2]) < 10.5).all()
    w4 = scenes.cluster_mixture(1000)
    assert w4.shape == (1000, 3)
    pos, rot = scenes.bspline_trajectory_batch(np.random.default_rng(4), 3)
    assert pos.shape == (192, 3) and rot.shape == (192, 3, 3)
    assert np.allclose(np.einsum("qji,qjk->qik", rot, rot), np.eye(3), atol=1e-12)


def test_c_abi_exports_every_declared_symbol():
    """libfif_b200.so loads without a GPU and exports every function include/fif_b200.h declares."""
    hdr = open(os.path.join(ROOT, "include", "fif_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(fif_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED)
    L = _lib.load()
    for name in declared:
        assert hasattr(L, name)
    assert L.fif_abi_version() == 2
    assert L.fif_build_scratch_bytes(1000) >= 1000 * 32


def test_c_abi_argument_errors_without_gpu():
    """Argument validation happens before any device work, so it runs on CPU."""
    L = _lib.load()
    m = _lib.Model()
    m.kind = 7
    st = L.fif_build(0, m, None, 0, None, None, 0, 1, None, 1.0, 0, None, None, None, None)
    assert st == -1 and b"model kind" in L.fif_last_error()
    st = L.fif_query(5, m, None, None, None, None, None, 1, 0, 0, *([None] * 8))
    assert st == -1
    with pytest.raises(_lib.FifCudaError):
        _lib.check(st, "fif_query")


def test_product_does_not_import_oracle():
    """The product package never reaches for the test oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2008_03324_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), fn
            assert "libfif_oracle" not in src, fn


def test_junction_basis_matches_reference():
    """planner.JunctionBasis restates traj._JunctionBasis (traj.py:50-89): Hermite maps,
    dynamic-cost forms and junction -> coefficient map against the reference's values."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "traj_opt.npz"))
    from paper_2008_03324_b200.planner import JunctionBasis

    b = JunctionBasis(g["durations"])
    for s in range(b.S):
        assert np.allclose(b.M[s], g["M"][s], rtol=1e-13, atol=1e-13)
    assert np.allclose(b.cost_matrix(4), g["R4"], rtol=1e-12, atol=1e-9)
    assert np.allclose(b.cost_matrix(2), g["R2"], rtol=1e-12, atol=1e-9)
    assert np.allclose(b.coeffs_from_derivs(g["D0"]), g["coeffs0"], rtol=1e-12, atol=1e-12)


def test_build_rows_rejects_non_float64_tensors():
    """The C ABI takes plain double pointers (include/fif_b200.h fif_build): a float32 landmark
    tensor would be reinterpreted, so the host refuses it before any library call."""
    import torch

    from paper_2008_03324_b200 import field as FD

    grid = F.GridConfig(np.zeros(3), 0.5, np.array([2, 2, 2]))
    with pytest.raises(TypeError):
        FD.build_rows(torch.zeros((4, 3), dtype=torch.float32), F.build_quad_model(), False, 1.0, torch.device("cpu"),
                      grid=grid)
    with pytest.raises(TypeError):
        FD.build_rows(torch.zeros((3, 4), dtype=torch.float64).t(), F.build_quad_model(), False, 1.0,
                      torch.device("cpu"), grid=grid)

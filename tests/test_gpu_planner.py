"""Planner-facing helpers: metric + analytic d/d[x,y,z,yaw] at
(position, yaw) states vs central differences of the oracle's metric, and the
trajectory information cost gradient vs finite differences."""
import numpy as np
import pytest

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import planner as P
from tests._helpers import models_from_golden, oracle_model
from tests.test_gpu_query import field_from_reference

pytestmark = pytest.mark.gpu


def _oracle_metric(oracle, g_small, grid, model, metric, pos, yaws, trilinear):
    slots = np.arange(grid.voxel_count, dtype=np.int32)
    v, st = oracle.metric_batch(slots, g_small[f"factors_{_name(model)}_info"], grid.origin, grid.voxel_size,
                                grid.dims, pos, np.ascontiguousarray(P.yaw_axes(yaws)), oracle_model(model), metric,
                                False, trilinear)
    return v, st


def _name(model):
    return "quad" if isinstance(model, F.QuadraticVisibility) else f"gp{model.n_v}"


@pytest.fixture(scope="module")
def setup(g_small, g_models):
    models = models_from_golden(g_models)
    grid = F.GridConfig(g_small["origin"], float(np.asarray(g_small["voxel_size"]).reshape(-1)[0]), g_small["dims"])
    return models, grid


@pytest.mark.parametrize("metric", ["det", "lmin", "trace"])
@pytest.mark.parametrize("mode", ["nearest", "trilinear"])
def test_metric_yaw_gradient(oracle, g_small, setup, metric, mode):
    models, grid = setup
    m = models["gp70"]
    f = field_from_reference(grid, m, "info", g_small["factors_gp70_info"])
    rng = np.random.default_rng(5)
    c = grid.centers()
    pos = rng.uniform(c[0], c[-1], size=(40, 3))
    g = (pos - grid.origin) / grid.voxel_size - (0.5 if mode == "trilinear" else 0.0)
    frac = g - np.floor(g)
    pos = pos[((frac > 1e-3) & (frac < 1 - 1e-3)).all(axis=1)]
    yaws = rng.uniform(-np.pi, np.pi, pos.shape[0])
    tri = mode == "trilinear"
    v, st = _oracle_metric(oracle, g_small, grid, m, metric, pos, yaws, tri)
    h = 1e-6
    fd = np.zeros((pos.shape[0], 4))
    for j in range(4):
        if j < 3:
            d = np.zeros(3)
            d[j] = h
            fd[:, j] = (_oracle_metric(oracle, g_small, grid, m, metric, pos + d, yaws, tri)[0] -
                        _oracle_metric(oracle, g_small, grid, m, metric, pos - d, yaws, tri)[0]) / (2 * h)
        else:
            fd[:, j] = (_oracle_metric(oracle, g_small, grid, m, metric, pos, yaws + h, tri)[0] -
                        _oracle_metric(oracle, g_small, grid, m, metric, pos, yaws - h, tri)[0]) / (2 * h)
    for f64 in (True, False):
        r = P.metric_yaw_batch(f, pos, yaws, metric, mode, grad=True, field_f64=f64)
        assert np.array_equal(r["in_field"], st == 0)
        assert np.allclose(r["values"], v, rtol=1e-4, atol=0)
        err = np.linalg.norm(r["grad"] - fd, axis=1) / np.maximum(np.linalg.norm(fd, axis=1), 1e-300)
        # lambda_min gradients always read the FP64 master (eigenvector sensitivity ~ 1/gap)
        tol = 1e-4
        print(f"[yaw {metric} {mode} f64={f64}] value {(np.abs(r['values'] - v) / np.abs(v)).max():.2e} grad {err.max():.2e}")
        assert err.max() <= tol, (f64, err.max())


def test_info_cost_gradient_and_gate(oracle, g_small, setup):
    models, grid = setup
    m = models["quad"]
    f = field_from_reference(grid, m, "info", g_small["factors_quad_info"])
    rng = np.random.default_rng(9)
    c = grid.centers()
    pos = rng.uniform(c[0], c[-1], size=(30, 3))
    yaws = rng.uniform(-np.pi, np.pi, 30)
    vals = P.metric_yaw_batch(f, pos, yaws, "det", "trilinear")["values"]
    pot = P.PotentialParams(epsilon=float(np.median(vals)), k_q=2.0)
    cost, g = P.info_cost_grad(f, pos, yaws, "det", pot, mu_v=0.7, dt=0.1, mode="trilinear")

    def total(p, y):
        v, st = _oracle_metric(oracle, g_small, grid, m, "det", p, y, True)
        return 0.7 * 0.1 * np.where(st == 0, P.info_potential(v, pot), pot.b_l).sum()

    assert cost == pytest.approx(total(pos, yaws), rel=1e-9)
    h = 1e-6
    for t in range(0, 30, 7):
        for j in range(4):
            pp, yp, pm, ym = pos.copy(), yaws.copy(), pos.copy(), yaws.copy()
            if j < 3:
                pp[t, j] += h
                pm[t, j] -= h
            else:
                yp[t] += h
                ym[t] -= h
            fd = (total(pp, yp) - total(pm, ym)) / (2 * h)
            assert g[t, j] == pytest.approx(fd, rel=1e-4, abs=1e-9 * max(1.0, abs(fd)))
    ok = P.gate_ok(f, pos, yaws, "det", pot.epsilon, "trilinear")
    assert np.array_equal(ok, vals >= pot.epsilon)


def test_poly_trajectory_gradient(oracle, g_small, setup):
    """Chain rule through the polynomial basis (traj.py:120-132) vs FD over the coefficients."""
    models, grid = setup
    m = models["quad"]
    f = field_from_reference(grid, m, "info", g_small["factors_quad_info"])
    rng = np.random.default_rng(13)
    c = grid.centers()
    lo, hi = c[0] + 0.3, c[-1] - 0.3
    S = 2
    coeffs = np.zeros((4, S, 8))
    for s in range(S):
        coeffs[:3, s, 0] = rng.uniform(lo, hi)
        coeffs[:3, s, 1] = rng.uniform(-0.2, 0.2, 3)
        coeffs[3, s, 0] = rng.uniform(-np.pi, np.pi)
        coeffs[3, s, 1] = rng.uniform(-0.5, 0.5)
    durations = np.array([1.0, 1.5])
    times = np.arange(0.0, 2.5, 0.1)
    vals = P.poly_eval(coeffs, durations, times)
    v0 = P.metric_yaw_batch(f, vals[:, :3], vals[:, 3], "det", "trilinear")["values"]
    pot = P.PotentialParams(epsilon=float(np.max(v0)) * 1.1, k_q=1.0)
    cost, grad = P.poly_info_cost_grad(f, coeffs, durations, times, "det", pot, mu_v=0.5, dt=0.1, mode="trilinear")

    def total(cf):
        vv = P.poly_eval(cf, durations, times)
        v, st = _oracle_metric(oracle, g_small, grid, m, "det", vv[:, :3], vv[:, 3], True)
        return 0.5 * 0.1 * np.where(st == 0, P.info_potential(v, pot), pot.b_l).sum()

    assert cost == pytest.approx(total(coeffs), rel=1e-9)
    h = 1e-6
    for (a, s, i) in [(0, 0, 0), (1, 1, 1), (2, 0, 2), (3, 1, 0), (3, 0, 3), (0, 1, 4)]:
        cp, cm = coeffs.copy(), coeffs.copy()
        cp[a, s, i] += h
        cm[a, s, i] -= h
        fd = (total(cp) - total(cm)) / (2 * h)
        assert grad[a, s, i] == pytest.approx(fd, rel=1e-4, abs=1e-9 * max(1.0, abs(fd)))


def test_traj_optimisation_replaces_fd_loop():
    """the reference's L-BFGS-B trajectory optimisation (traj.optimize_trajectory,
    traj.py:411-463, central-difference gradients: 2 x n_free cost evaluations per gradient)
    driven instead by the analytic pose gradient of a GPU field.  Same problem as the golden
    run of the reference (quad info field, trilinear det metric, tests/golden/traj_opt.npz):
    the initial cost matches the reference's, the analytic gradient matches central
    differences, and L-BFGS-B reaches at least the reference's final cost with a small
    fraction of its batched field evaluations."""
    import os

    from paper_2008_03324_b200.planner import InfoTrajectoryProblem, PotentialParams, optimize_info_trajectory

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "traj_opt.npz"))
    grid = F.GridConfig(g["origin"], g["voxel_size"][0], g["dims"])
    fld = F.Field.build(g["points"], grid, F.build_quad_model(), "info", exact=True)
    prob = InfoTrajectoryProblem(g["D0"], g["durations"], fld, PotentialParams(float(g["epsilon"][0])), metric="det",
                                 mode="trilinear", mu_d=float(g["mu_d"][0]), mu_v=float(g["mu_v"][0]),
                                 dt=float(g["dt"][0]))
    x0 = prob.x0()
    c0 = prob.cost(x0)
    assert abs(c0 - g["initial_cost"][0]) <= 1e-9 * g["initial_cost"][0]
    ga, gf = prob.gradient(x0), prob.gradient_fd(x0)
    rel = np.linalg.norm(ga - gf) / np.linalg.norm(gf)
    res = optimize_info_trajectory(prob, "analytic", max_iters=25)
    ref_final, ref_evals = float(g["final_cost"][0]), int(g["n_evals"][0])
    print(f"analytic vs FD gradient at x0: {rel:.2e}; reference (FD) {g['initial_cost'][0]:.4e} -> {ref_final:.4e} in "
          f"{ref_evals} evaluations; ours (analytic) -> {res['cost']:.4e} in {res['n_evals']} evaluations, "
          f"{res['iterations']} iterations, {res['seconds']:.2f} s")
    assert rel <= 1e-3
    assert res["cost"] <= ref_final * 1.02
    assert res["n_evals"] * 20 <= ref_evals

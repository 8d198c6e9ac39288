"""Planner-facing batch evaluation over a GPU field.

The reference planners evaluate the information metric of (position, yaw) states
through `rrt._info_values` (rrt.py:88-96) and differentiate the trajectory cost by
central differences (`traj._FreeParamProblem.gradient`, traj.py:383-398: two cost
evaluations per free parameter).  These helpers return the same values from one
batched GPU query together with the analytic derivatives w.r.t. position and yaw
(A15 and the det / lambda_min gradients of fif_query_ex), so a planner replaces its
finite differences by one chain rule: d cost / d x = sum_t J_t^T g_t with
J_t = d(position_t, yaw_t)/dx from its polynomial basis (traj.py:120-132).

Camera convention (rrt.py:23-35): heading-mounted camera, R = Rz(yaw) R_CAM_MOUNT,
optical axis (cos yaw, sin yaw, 0).  A yaw step is the world-frame rotation about
e_z, so d q / d yaw = e_z . d q / d theta.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from .errors import WrongFactorKind
from .field import Field
from .fim import DEFAULT_SIGMA, METRICS, PinholeCamera, pc_metric_yaw_batch_device
from .scenes import R_CAM_MOUNT, yaw_rotation

__all__ = ["R_CAM_MOUNT", "yaw_rotation", "ExactInfoRepr", "yaw_axes", "metric_yaw_batch", "gate_ok",
           "PotentialParams", "info_potential", "info_potential_grad", "JunctionBasis", "InfoTrajectoryProblem",
           "optimize_info_trajectory",
           "info_cost_grad", "poly_eval", "poly_info_cost_grad"]


class ExactInfoRepr:
    """Information evaluation against the raw landmark set (rrt.py:54-71) on the GPU:
    `metric_batch(positions, yaws, metric)` runs fif_pc_metric_yaw (the point-cloud 6x6 of
    each yaw pose, then det / lmin / trace), the planners' exact comparator for a field."""

    def __init__(self, points, camera: PinholeCamera | None = None, sigma: float = DEFAULT_SIGMA, device=None):
        self.points = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
        self.camera = camera if camera is not None else PinholeCamera.from_fov()
        self.sigma = float(sigma)
        self.device = _device.require_cuda(device)
        self._pts = _device.to_device_f64(self.points, self.device, (3,))

    def metric_batch(self, positions, yaws, metric: str):
        if metric not in METRICS:
            raise ValueError(f"unknown metric {metric!r}")
        pos = _device.to_device_f64(positions, self.device, (3,))
        vals = pc_metric_yaw_batch_device(pos, np.asarray(yaws, dtype=np.float64).reshape(-1), self._pts,
                                          self.camera, self.sigma, R_CAM_MOUNT, metric)
        v = _device.to_numpy(vals)
        return v, np.ones(len(v), dtype=bool)


def yaw_axes(yaws) -> np.ndarray:
    """Optical axes (cos, sin, 0) of a heading-mounted camera (rrt.py:32-35)."""
    yaws = np.asarray(yaws, dtype=np.float64)
    return np.stack([np.cos(yaws), np.sin(yaws), np.zeros_like(yaws)], axis=-1)


def metric_yaw_batch(field: Field, positions, yaws, metric: str = "det", mode: str = "nearest",
                     grad: bool = False, field_f64: bool = False) -> dict:
    """Metric at (position, yaw) states, as `field.metric_axis_batch(positions,
    yaw_axes(yaws), metric, mode)` (rrt.py:96), plus with grad=True its derivatives
    (Q, 4) = d/d[x, y, z, yaw].  Returns numpy arrays: values, in_field[, grad].
    field_f64 selects the FP64 master of a GP field instead of its FP32 copy."""
    if metric not in ("det", "lmin", "trace"):
        raise ValueError(f"unknown metric {metric!r}")
    if metric != "trace" and field.factor_kind != "info":
        raise WrongFactorKind("det/lmin require an info-factor field")
    dev = field.device
    pos = _device.to_device_f64(positions, dev, (3,))
    ax = torch.from_numpy(np.ascontiguousarray(yaw_axes(yaws).reshape(-1, 3))).to(dev)
    res = field.query_device(pos, ax, mode, trace=metric == "trace", det=metric == "det", lmin=metric == "lmin",
                             grad=grad, field_f64=field_f64)
    out = {"values": _device.to_numpy(res[metric]), "in_field": _device.to_numpy(res["status"] == 0)}
    if grad:
        g6 = _device.to_numpy(res[f"{metric}_grad"])
        out["grad"] = np.concatenate([g6[:, :3], g6[:, 5:6]], axis=1)  # d/dt, e_z . d/dtheta
    return out


def gate_ok(field: Field, positions, yaws, metric: str, threshold: float, mode: str = "nearest") -> np.ndarray:
    """Information gate of `rrt.state_valid` (rrt.py:99-111) for a batch: in field and
    metric >= threshold (out of field counts as invalid)."""
    r = metric_yaw_batch(field, positions, yaws, metric, mode)
    return r["in_field"] & (r["values"] >= threshold)


@dataclass(frozen=True)
class PotentialParams:
    """Piecewise information potential (costs.py:58-77); k_l, b_l keep it C1 at v = 0."""

    epsilon: float
    k_q: float = 1.0

    def __post_init__(self) -> None:
        if self.epsilon < 0:
            raise ValueError("epsilon must be non-negative")
        if self.k_q <= 0:
            raise ValueError("k_q must be positive")

    @property
    def k_l(self) -> float:
        return -2.0 * self.k_q * self.epsilon

    @property
    def b_l(self) -> float:
        return self.k_q * self.epsilon ** 2


def info_potential(v, p: PotentialParams):
    """costs.py:79-85."""
    a = np.asarray(v, dtype=np.float64)
    return np.where(a > p.epsilon, 0.0, np.where(a >= 0.0, p.k_q * (a - p.epsilon) ** 2, p.k_l * a + p.b_l))


def info_potential_grad(v, p: PotentialParams):
    """costs.py:88-93."""
    a = np.asarray(v, dtype=np.float64)
    return np.where(a > p.epsilon, 0.0, np.where(a >= 0.0, 2.0 * p.k_q * (a - p.epsilon), p.k_l))


def info_cost_grad(field: Field, positions, yaws, metric: str, potential: PotentialParams, mu_v: float, dt: float,
                   mode: str = "nearest"):
    """Information term of the sampled trajectory cost (traj.py:357-363) and its
    gradient w.r.t. every sample's (x, y, z, yaw): cost = mu_v dt sum_t pot(v_t), with
    out-of-field samples charged b_l (zero gradient).  Returns (cost, grad (T, 4))."""
    r = metric_yaw_batch(field, positions, yaws, metric, mode, grad=True)
    v, ok = r["values"], r["in_field"]
    pot = np.where(ok, info_potential(v, potential), potential.b_l)
    dpot = np.where(ok, info_potential_grad(v, potential), 0.0)
    cost = float(mu_v * pot.sum() * dt)
    return cost, (mu_v * dt) * dpot[:, None] * r["grad"]


def _poly_locate(durations: np.ndarray, times: np.ndarray):
    """Segment index and local time of each sample (traj.py:113-118, PolyTrajectory._locate)."""
    ends = np.cumsum(durations)
    seg = np.minimum(np.searchsorted(ends, times, side="right"), len(durations) - 1)
    return seg, times - (ends - durations)[seg]


def poly_eval(coeffs, durations, times) -> np.ndarray:
    """(K, 4) x, y, z, yaw of a piecewise polynomial with ascending-power coefficients
    (4, S, 8) (PolyTrajectory.eval, traj.py:120-132, order 0)."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    times = np.atleast_1d(np.asarray(times, dtype=np.float64))
    seg, tau = _poly_locate(np.asarray(durations, dtype=np.float64).reshape(-1), times)
    basis = tau[:, None] ** np.arange(8)[None, :]
    return np.einsum("ki,aki->ka", basis, coeffs[:, seg, :])


def poly_info_cost_grad(field: Field, coeffs, durations, times, metric: str, potential: PotentialParams, mu_v: float,
                        dt: float, mode: str = "nearest"):
    """Information term of the sampled trajectory cost (traj.py:350-365) for a
    PolyTrajectory given by its coefficients, and its exact gradient w.r.t. the
    coefficients (4, S, 8): the chain rule through the power basis that replaces the
    central differences of traj._FreeParamProblem.gradient (traj.py:383-398) for this
    term.  Returns (cost, d cost / d coeffs)."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    durations = np.asarray(durations, dtype=np.float64).reshape(-1)
    times = np.atleast_1d(np.asarray(times, dtype=np.float64))
    vals = poly_eval(coeffs, durations, times)
    cost, g = info_cost_grad(field, vals[:, :3], vals[:, 3], metric, potential, mu_v, dt, mode)
    seg, tau = _poly_locate(durations, times)
    basis = tau[:, None] ** np.arange(8)[None, :]
    grad = np.zeros_like(coeffs)
    for a in range(4):
        np.add.at(grad[a], seg, g[:, a:a + 1] * basis)
    return cost, grad


# ── trajectory optimisation with the analytic information gradient ─────────
# The reference optimises the free junction derivatives of a piecewise polynomial with
# L-BFGS-B (traj.optimize_trajectory, traj.py:411-463); its gradient of the sampled cost is
# a central difference per free parameter (traj._FreeParamProblem.gradient, traj.py:383-398:
# 2 x n_free cost evaluations, each a batched metric query).  InfoTrajectoryProblem keeps the
# reference's parametrisation and cost (dynamic term + information potential; the obstacle
# term is out of scope here) and differentiates the information term analytically: one
# batched GPU query with pose gradients, chained through the (linear) junction -> coefficient
# -> sample maps.

NDERIV = 4  # junction continuity: value + derivatives 1..3 (traj.py:27)


def _hermite_matrix(T: float) -> np.ndarray:
    """Coefficients (ascending powers 0..7) -> derivatives 0..3 at both ends of [0, T]."""
    import math

    A = np.zeros((8, 8))
    for k in range(NDERIV):
        A[k, k] = math.factorial(k)
        for i in range(k, 8):
            A[NDERIV + k, i] = math.perm(i, k) * T ** (i - k)
    return A


def _deriv_gram(T: float, k: int) -> np.ndarray:
    """Q with c^T Q c = integral over [0, T] of the squared k-th derivative."""
    import math

    Q = np.zeros((8, 8))
    for i in range(k, 8):
        for j in range(k, 8):
            p = i + j - 2 * k + 1
            Q[i, j] = math.perm(i, k) * math.perm(j, k) * T ** p / p
    return Q


class JunctionBasis:
    """Linear maps between stacked junction derivatives D (per axis, length 4 (S + 1)) and
    per-segment coefficients, and the quadratic dynamic-cost forms (traj.py:50-89)."""

    def __init__(self, durations):
        self.durations = np.asarray(durations, dtype=np.float64).reshape(-1)
        if (self.durations <= 0).any() or not np.isfinite(self.durations).all():
            raise ValueError("segment durations must be positive and finite")
        self.S = len(self.durations)
        self.L = NDERIV * (self.S + 1)
        self.M = [np.linalg.inv(_hermite_matrix(T)) for T in self.durations]

    def cost_matrix(self, order: int) -> np.ndarray:
        R = np.zeros((self.L, self.L))
        for s, T in enumerate(self.durations):
            i = NDERIV * s
            R[i:i + 8, i:i + 8] += self.M[s].T @ _deriv_gram(T, order) @ self.M[s]
        return R

    def coeffs_from_derivs(self, D: np.ndarray) -> np.ndarray:
        """D (..., L) -> coefficients (..., S, 8)."""
        D = np.asarray(D, dtype=np.float64)
        out = np.empty(D.shape[:-1] + (self.S, 8))
        for s in range(self.S):
            out[..., s, :] = D[..., NDERIV * s:NDERIV * s + 8] @ self.M[s].T
        return out

    def derivs_grad_from_coeffs_grad(self, G: np.ndarray) -> np.ndarray:
        """Adjoint of coeffs_from_derivs: d cost / d coeffs (..., S, 8) -> d cost / d D (..., L)."""
        out = np.zeros(G.shape[:-2] + (self.L,))
        for s in range(self.S):
            out[..., NDERIV * s:NDERIV * s + 8] += G[..., s, :] @ self.M[s]
        return out


class InfoTrajectoryProblem:
    """traj._FreeParamProblem (traj.py:308-398) over a GPU field: free parameters are the
    derivatives 0..3 of every axis at the internal junctions; cost = mu_d sum_axes D^T R D
    (snap for x, y, z, yaw acceleration) + mu_v dt sum_t pot(metric(state_t)).
    `gradient` is analytic (one batched query); `gradient_fd` is the reference's central
    difference (2 x n_free sampled-cost evaluations), kept for comparison."""

    def __init__(self, D0, durations, field: Field, potential: PotentialParams, metric: str = "det",
                 mode: str = "trilinear", mu_d: float = 1.0, mu_v: float = 1.0, dt: float = 0.1,
                 fd_step: float = 1e-4):
        self.basis = JunctionBasis(durations)
        self.D0 = np.asarray(D0, dtype=np.float64).reshape(4, self.basis.L).copy()
        self.free_idx = np.arange(NDERIV, self.basis.L - NDERIV)
        self.field, self.potential, self.metric, self.mode = field, potential, metric, mode
        self.mu_d, self.mu_v, self.dt, self.fd_step = mu_d, mu_v, dt, fd_step
        self.R = [self.basis.cost_matrix(4), self.basis.cost_matrix(2)]
        k = max(1, int(round(float(self.basis.durations.sum()) / dt)))
        self.times = np.arange(k) * dt
        self.n_evals = 0  # sampled-cost evaluations (batched field queries), as the reference counts them

    def x0(self) -> np.ndarray:
        return self.D0[:, self.free_idx].reshape(-1).copy()

    def derivs(self, x) -> np.ndarray:
        D = self.D0.copy()
        D[:, self.free_idx] = np.asarray(x, dtype=np.float64).reshape(4, -1)
        return D

    def coeffs(self, x) -> np.ndarray:
        return self.basis.coeffs_from_derivs(self.derivs(x))

    def _dynamic(self, D):
        cost, grad = 0.0, np.zeros_like(D)
        for a in range(4):
            RD = self.R[0 if a < 3 else 1] @ D[a]
            cost += float(D[a] @ RD)
            grad[a] = 2.0 * RD
        return self.mu_d * cost, self.mu_d * grad

    def _sampled(self, coeffs, with_grad: bool):
        self.n_evals += 1
        if with_grad:
            return poly_info_cost_grad(self.field, coeffs, self.basis.durations, self.times, self.metric,
                                       self.potential, self.mu_v, self.dt, self.mode)
        vals = poly_eval(coeffs, self.basis.durations, self.times)
        r = metric_yaw_batch(self.field, vals[:, :3], vals[:, 3], self.metric, self.mode)
        pot = np.where(r["in_field"], info_potential(r["values"], self.potential), self.potential.b_l)
        return float(self.mu_v * pot.sum() * self.dt), None

    def cost(self, x) -> float:
        D = self.derivs(x)
        return self._dynamic(D)[0] + self._sampled(self.basis.coeffs_from_derivs(D), False)[0]

    def cost_and_gradient(self, x):
        D = self.derivs(x)
        dc, dg = self._dynamic(D)
        sc, sg = self._sampled(self.basis.coeffs_from_derivs(D), True)
        g = dg + self.basis.derivs_grad_from_coeffs_grad(sg)
        return dc + sc, g[:, self.free_idx].reshape(-1)

    def gradient(self, x) -> np.ndarray:
        return self.cost_and_gradient(x)[1]

    def gradient_fd(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        D = self.derivs(x)
        g = self._dynamic(D)[1][:, self.free_idx].reshape(-1)
        h = self.fd_step
        for i in range(x.size):
            xp = x.copy()
            xp[i] += h
            cp = self._sampled(self.coeffs(xp), False)[0]
            xp[i] -= 2 * h
            cm = self._sampled(self.coeffs(xp), False)[0]
            g[i] += (cp - cm) / (2 * h)
        return g


def optimize_info_trajectory(problem: InfoTrajectoryProblem, gradient: str = "analytic", max_iters: int = 100):
    """L-BFGS-B over the free junction derivatives, tracking the best iterate
    (traj.optimize_trajectory, traj.py:411-463).  gradient = "analytic" (cost and gradient
    from one batched query per evaluation) or "fd" (the reference's central differences).
    Returns dict(x, cost, initial_cost, iterations, n_evals, seconds)."""
    import time

    from scipy.optimize import minimize

    x0 = problem.x0()
    problem.n_evals = 0
    c0 = problem.cost(x0)
    best = {"x": x0.copy(), "cost": c0}
    iters = 0

    def track(x, c):
        if c < best["cost"]:
            best["cost"], best["x"] = c, np.array(x, copy=True)

    def cb(_xk):
        nonlocal iters
        iters += 1

    t0 = time.perf_counter()
    if gradient == "analytic":
        def fun(x):
            c, g = problem.cost_and_gradient(x)
            track(x, c)
            return c, g

        minimize(fun, x0, jac=True, method="L-BFGS-B", callback=cb, options={"maxiter": max_iters})
    elif gradient == "fd":
        def fun(x):
            c = problem.cost(x)
            track(x, c)
            return c

        minimize(fun, x0, jac=problem.gradient_fd, method="L-BFGS-B", callback=cb, options={"maxiter": max_iters})
    else:
        raise ValueError("gradient must be 'analytic' or 'fd'")
    return {"x": best["x"], "cost": best["cost"], "initial_cost": c0, "iterations": iters,
            "n_evals": problem.n_evals, "seconds": time.perf_counter() - t0}

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
           "PotentialParams", "info_potential", "info_potential_grad",
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

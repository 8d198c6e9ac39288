"""Per-landmark and per-pose Fisher information (mirrors fifield/fim.py).

The per-landmark helpers are O(1) host math; `exact_pose_fim(_batch)` — the
paper's point-cloud comparison method — runs on the GPU (fif_pc_fim).
Bearing model with world-side pose perturbation, state [translation; rotation]:
I_i = (1/sigma^2) [-I3, skew(p)]^T (I3 - u u^T)/n^2 [-I3, skew(p)]  (fim.py:1-11).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import DegeneratePoint
from .geometry import Pose, skew

DEFAULT_SIGMA = 1.0
METRICS = ("det", "lmin", "trace")
_RANGE_EPS = 1e-9


@dataclass(frozen=True)
class PinholeCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    half_fov_alpha: float

    def __post_init__(self) -> None:
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0.0 < self.half_fov_alpha < np.pi):
            raise ValueError("half_fov_alpha must be in (0, pi)")

    @staticmethod
    def from_fov(horizontal_fov: float = np.pi / 2, width: int = 640, height: int = 640) -> "PinholeCamera":
        f = 0.5 * width / np.tan(0.5 * horizontal_fov)
        return PinholeCamera(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, width=width, height=height,
                             half_fov_alpha=horizontal_fov / 2.0)

    def as_tuple(self) -> tuple[float, float, float, float, float, float]:
        return (float(self.fx), float(self.fy), float(self.cx), float(self.cy), float(self.width),
                float(self.height))


def _block(p: np.ndarray, t: np.ndarray, sigma: float) -> np.ndarray:
    d = p - t
    n2 = float(d @ d)
    u = d / np.sqrt(n2)
    w = 1.0 / (sigma * sigma * n2)
    c2 = np.cross(p, u)
    s = skew(p)
    top_left = w * (np.eye(3) - np.outer(u, u))
    top_right = -w * (s + np.outer(u, c2))
    bottom_right = w * (float(p @ p) * np.eye(3) - np.outer(p, p) - np.outer(c2, c2))
    return np.block([[top_left, top_right], [top_right.T, bottom_right]])


def bearing_jacobian(pose: Pose, landmark_position) -> np.ndarray:
    """3x6 d bearing / d [t; theta] for the world-side perturbation."""
    p = np.asarray(landmark_position, dtype=np.float64)
    d = p - pose.translation
    n = np.linalg.norm(d)
    if n <= _RANGE_EPS:
        raise DegeneratePoint(f"landmark range {n:.3e} below threshold")
    pc = pose.rotation.T @ d
    proj = np.eye(3) / n - np.outer(pc, pc) / n ** 3
    return proj @ pose.rotation.T @ np.hstack([-np.eye(3), skew(p)])


def landmark_fim(camera_position, landmark_position, sigma: float = DEFAULT_SIGMA) -> np.ndarray:
    t = np.asarray(camera_position, dtype=np.float64)
    p = np.asarray(landmark_position, dtype=np.float64)
    n = np.linalg.norm(p - t)
    if n <= _RANGE_EPS:
        raise DegeneratePoint(f"landmark range {n:.3e} below threshold")
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    return _block(p, t, sigma)


def exact_visible(pose: Pose, landmark_position, camera: PinholeCamera) -> bool:
    pc = pose.rotation.T @ (np.asarray(landmark_position, dtype=np.float64) - pose.translation)
    z = pc[2]
    if z <= 0.0:
        return False
    u = camera.fx * pc[0] / z + camera.cx
    v = camera.fy * pc[1] / z + camera.cy
    return bool(0.0 <= u < camera.width and 0.0 <= v < camera.height)


def exact_pose_fim_batch_device(rotations: torch.Tensor, translations: torch.Tensor, landmarks: torch.Tensor,
                                camera: PinholeCamera, sigma: float = DEFAULT_SIGMA, mask: torch.Tensor | None = None,
                                out: torch.Tensor | None = None) -> torch.Tensor:
    """Device-resident entry point: (Q,9)/(Q,3,3) R, (Q,3) t, (N,3) p float64 CUDA tensors -> (Q,36) f64."""
    dev = rotations.device
    q = translations.shape[0]
    if out is None:
        out = torch.empty((q, 36), dtype=torch.float64, device=dev)
    cam = _lib.make_camera(camera.as_tuple())
    with torch.cuda.device(dev):
        _lib.check(_lib.load().fif_pc_fim(_lib.ptr(rotations), _lib.ptr(translations), q, _lib.ptr(landmarks),
                                          landmarks.shape[0], cam, float(sigma), _lib.ptr(out), _lib.ptr(mask),
                                          _device.stream_handle(dev)), "fif_pc_fim")
    return out


def exact_pose_fim_batch(rotations, translations, landmark_positions, camera: PinholeCamera,
                         sigma: float = DEFAULT_SIGMA) -> np.ndarray:
    """(Q,6,6) exact FIMs for Q poses (fim.py:132-146), computed on the GPU."""
    dev = _device.require_cuda()
    r = _device.to_device_f64(rotations, dev, (9,))
    t = _device.to_device_f64(translations, dev, (3,))
    p = _device.to_device_f64(landmark_positions, dev, (3,))
    out = exact_pose_fim_batch_device(r, t, p, camera, sigma)
    return _device.to_numpy(out).reshape(-1, 6, 6)


def pc_metric_yaw_batch_device(positions: torch.Tensor, yaws, landmarks: torch.Tensor, camera: PinholeCamera,
                               sigma: float, r_base, metric: str, out: torch.Tensor | None = None,
                               fim: torch.Tensor | None = None, mask: torch.Tensor | None = None) -> torch.Tensor:
    """Exact point-cloud metric at yaw-only poses on the device (kernels.pc_metric_yaw_batch,
    kernels.py:1599-1606 -> _nb_pc_metric_yaw_batch 611-625): R = Rz(yaw) r_base in the
    reference's operation order, the point-cloud 6x6, then det / lmin / trace.  cos / sin of
    the yaws are taken on the host with numpy, as the reference does."""
    if metric not in _lib.METRIC_IDS:
        raise ValueError(f"unknown metric {metric!r}; expected one of {METRICS}")
    dev = positions.device
    q = positions.shape[0]
    y = np.asarray(yaws.cpu().numpy() if isinstance(yaws, torch.Tensor) else yaws, dtype=np.float64).reshape(-1)
    if y.shape[0] != q:
        raise ValueError("positions and yaws must have the same length")
    cs = torch.from_numpy(np.ascontiguousarray(np.stack([np.cos(y), np.sin(y)], axis=1))).to(dev)
    rb = (ctypes.c_double * 9)(*np.asarray(r_base, dtype=np.float64).reshape(9).tolist())
    if out is None:
        out = torch.empty(q, dtype=torch.float64, device=dev)
    cam = _lib.make_camera(camera.as_tuple())
    with torch.cuda.device(dev):
        _lib.check(_lib.load().fif_pc_metric_yaw(_lib.ptr(positions), _lib.ptr(cs), q, _lib.ptr(landmarks),
                                                 landmarks.shape[0], cam, float(sigma), ctypes.byref(rb),
                                                 _lib.METRIC_IDS[metric], _lib.ptr(out), _lib.ptr(fim), _lib.ptr(mask),
                                                 _device.stream_handle(dev)), "fif_pc_metric_yaw")
    return out


def pc_metric_yaw_batch(positions, yaws, landmark_positions, camera: PinholeCamera, sigma: float, r_base,
                        metric: str) -> np.ndarray:
    """Host-array front end of pc_metric_yaw_batch_device (the reference kernel boundary's
    pc_metric_yaw_batch(positions, yaws, points, cam, sigma, r_base, mid))."""
    dev = _device.require_cuda()
    pos = _device.to_device_f64(positions, dev, (3,))
    pts = _device.to_device_f64(landmark_positions, dev, (3,))
    return _device.to_numpy(pc_metric_yaw_batch_device(pos, yaws, pts, camera, sigma, r_base, metric))


def exact_pose_fim(pose: Pose, landmark_positions, camera: PinholeCamera, sigma: float = DEFAULT_SIGMA) -> np.ndarray:
    pts = np.asarray(landmark_positions, dtype=np.float64).reshape(-1, 3)
    if pts.size == 0:
        return np.zeros((6, 6))
    return exact_pose_fim_batch(pose.rotation[None], pose.translation[None], pts, camera, sigma)[0]


def fim_metric(fim, kind: str) -> float:
    if kind not in METRICS:
        raise ValueError(f"unknown metric {kind!r}; expected one of {METRICS}")
    m = np.asarray(fim, dtype=np.float64)
    if kind == "det":
        return float(np.linalg.det(m))
    if kind == "lmin":
        return float(np.linalg.eigvalsh(m)[0])
    return float(np.trace(m))

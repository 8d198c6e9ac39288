"""Landmark scenes and the seeded synthetic workloads of BASELINE.json's configs.

Scene / gen_uniform / gen_clustered mirror fifield/scenes.py:15-111 (JSONL I/O,
box-uniform and clipped-cluster generators).  The config_* generators build the
five benchmark workloads exactly as SURVEY.md §8(d) fixes them (all RNG is
numpy.random.default_rng(seed); the seeds are part of the config).  They stand
in for the paper's SfM maps, which are not available (no dataset is shipped).
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .geometry import rot_z

R_CAM_MOUNT = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])  # rrt.py:25


@dataclass
class Scene:
    positions: np.ndarray
    view_dirs: np.ndarray | None = None
    ids: np.ndarray | None = None

    def __post_init__(self) -> None:
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1, 3)
        if self.view_dirs is not None:
            self.view_dirs = np.ascontiguousarray(self.view_dirs, dtype=np.float64).reshape(-1, 3)
            if self.view_dirs.shape[0] != self.positions.shape[0]:
                raise ValueError("view_dirs count does not match positions")
        self.ids = (np.arange(self.positions.shape[0], dtype=np.int64) if self.ids is None
                    else np.asarray(self.ids, dtype=np.int64).reshape(-1))

    @property
    def count(self) -> int:
        return self.positions.shape[0]

    def save(self, path) -> None:
        with open(path, "w") as f:
            for i in range(self.count):
                rec = {"id": int(self.ids[i]), "p": self.positions[i].tolist()}
                if self.view_dirs is not None:
                    rec["view_dir"] = self.view_dirs[i].tolist()
                f.write(json.dumps(rec) + "\n")

    @staticmethod
    def load(path) -> "Scene":
        ids, pts, dirs, any_dir = [], [], [], False
        with open(path) as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                rec = json.loads(line)
                ids.append(int(rec["id"]))
                pts.append([float(v) for v in rec["p"]])
                vd = rec.get("view_dir")
                any_dir |= vd is not None
                dirs.append([float(v) for v in vd] if vd is not None else [0.0, 0.0, 0.0])
        return Scene(np.asarray(pts, dtype=np.float64).reshape(-1, 3),
                     np.asarray(dirs, dtype=np.float64) if any_dir else None, np.asarray(ids, dtype=np.int64))


def _unit_rows(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def gen_uniform(count, lo=(-5.0, -5.0, 0.0), hi=(5.0, 5.0, 5.0), seed=0, with_view_dirs=False) -> Scene:
    rng = np.random.default_rng(seed)
    pos = rng.uniform(np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64), size=(count, 3))
    return Scene(pos, _unit_rows(rng, count) if with_view_dirs else None)


def gen_clustered(count, n_clusters=6, spread=0.6, lo=(-5.0, -5.0, 0.0), hi=(5.0, 5.0, 5.0), seed=0,
                  with_view_dirs=False) -> Scene:
    rng = np.random.default_rng(seed)
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    pad = np.minimum(spread, (hi - lo) / 4)
    centres = rng.uniform(lo + pad, hi - pad, size=(n_clusters, 3))
    which = rng.integers(0, n_clusters, size=count)
    pos = np.clip(centres[which] + rng.normal(scale=spread, size=(count, 3)), lo, hi)
    return Scene(pos, _unit_rows(rng, count) if with_view_dirs else None)


# ── batched pose helpers ────────────────────────────────────────────
def quat_to_rot(q: np.ndarray) -> np.ndarray:
    """(n,4) (w,x,y,z) -> (n,3,3), same formula as geometry.random_rotation."""
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    r = np.empty((q.shape[0], 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def uniform_rotations(rng, n) -> np.ndarray:
    return quat_to_rot(rng.standard_normal((n, 4)))


def ypr_rotations(yaw, pitch, roll) -> np.ndarray:
    """R = Rz(yaw) Ry(pitch) Rx(roll) for arrays of angles."""
    cy, sy, cp, sp, cr, sr = np.cos(yaw), np.sin(yaw), np.cos(pitch), np.sin(pitch), np.cos(roll), np.sin(roll)
    r = np.empty((np.size(yaw), 3, 3))
    r[:, 0, 0] = cy * cp
    r[:, 0, 1] = cy * sp * sr - sy * cr
    r[:, 0, 2] = cy * sp * cr + sy * sr
    r[:, 1, 0] = sy * cp
    r[:, 1, 1] = sy * sp * sr + cy * cr
    r[:, 1, 2] = sy * sp * cr - cy * sr
    r[:, 2, 0] = -sp
    r[:, 2, 1] = cp * sr
    r[:, 2, 2] = cp * cr
    return r


# ── the five BASELINE.json workloads ───────────────
@dataclass
class Workload:
    name: str
    points: np.ndarray
    grid: tuple           # (origin, voxel_size, dims)
    positions: np.ndarray | None = None
    rotations: np.ndarray | None = None


def config1(n_queries: int = 1000) -> Workload:
    """2 000 uniform landmarks in [-5,5]^2 x [0,3] (seed 0); grid 21x21x7 @ 0.5 m."""
    pts = gen_uniform(2000, lo=(-5.0, -5.0, 0.0), hi=(5.0, 5.0, 3.0), seed=0).positions
    grid = (np.array([-5.25, -5.25, -0.25]), 0.5, np.array([21, 21, 7]))
    pos, rots = _interior_queries(grid, n_queries, seed=1)
    return Workload("config1", pts, grid, pos, rots)


def room_walls(n: int = 20000, seed: int = 0, half: float = 10.0, height: float = 5.0, noise: float = 0.05):
    """Landmarks on the floor and 4 walls of a [-h,h]^2 x [0,H] room, area-proportional
    (floor 1/2, each wall 1/8 for h=10, H=5), N(0, noise) along the surface normal; float32."""
    rng = np.random.default_rng(seed)
    a_floor, a_wall = (2 * half) ** 2, 2 * half * height
    total = a_floor + 4 * a_wall
    n_floor = int(round(n * a_floor / total))
    n_wall = [(n - n_floor) // 4 + (1 if k < (n - n_floor) % 4 else 0) for k in range(4)]
    parts = []
    f = np.column_stack([rng.uniform(-half, half, n_floor), rng.uniform(-half, half, n_floor),
                         rng.normal(0.0, noise, n_floor)])
    parts.append(f)
    for k, m in enumerate(n_wall):
        s = rng.uniform(-half, half, m)
        h = rng.uniform(0.0, height, m)
        off = rng.normal(0.0, noise, m)
        if k == 0:
            w = np.column_stack([s, np.full(m, -half) + off, h])
        elif k == 1:
            w = np.column_stack([s, np.full(m, half) + off, h])
        elif k == 2:
            w = np.column_stack([np.full(m, -half) + off, s, h])
        else:
            w = np.column_stack([np.full(m, half) + off, s, h])
        parts.append(w)
    return np.vstack(parts).astype(np.float32).astype(np.float64)


def _interior_queries(grid, n, seed):
    origin, vs, dims = grid
    first = origin + 0.5 * vs
    last = origin + (np.asarray(dims) - 0.5) * vs
    rng = np.random.default_rng(seed)
    pos = rng.uniform(first, last, size=(n, 3))
    return pos, uniform_rotations(rng, n)


def config2(n_queries: int = 100000) -> Workload:
    """20 000 float32 room landmarks; grid 81x81x21 @ 0.25 m; full 6x6 + gradient queries."""
    pts = room_walls(20000, seed=0)
    grid = (np.array([-10.125, -10.125, -0.125]), 0.25, np.array([81, 81, 21]))
    pos, rots = _interior_queries(grid, n_queries, seed=1)
    return Workload("config2", pts, grid, pos, rots)


def config3(n_poses: int = 1000000) -> Workload:
    """Point-cloud baseline: config-2 landmarks, poses U([-10,10]^2 x [0,5]) x uniform SO(3) (seed 2)."""
    w2 = config2(0)
    rng = np.random.default_rng(2)
    pos = rng.uniform([-10.0, -10.0, 0.0], [10.0, 10.0, 5.0], size=(n_poses, 3))
    return Workload("config3", w2.points, w2.grid, pos, uniform_rotations(rng, n_poses))


def cluster_mixture(n: int = 1000000, k: int = 64, seed: int = 3, lo=(-50.0, -50.0, 0.0), hi=(50.0, 50.0, 20.0)):
    """Mixture of k isotropic Gaussians: centres U(box), sigma_c ~ U[0.5, 3] m, uniform assignment; float32."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(lo, hi, size=(k, 3))
    sig = rng.uniform(0.5, 3.0, size=k)
    which = rng.integers(0, k, size=n)
    pts = centres[which] + rng.standard_normal((n, 3)) * sig[which, None]
    return pts.astype(np.float32).astype(np.float64)


def config4(kind: str = "trace", n_points: int = 1000000) -> Workload:
    pts = cluster_mixture(n_points)
    if kind == "trace":
        grid = (np.array([-50.1, -50.1, -0.1]), 0.2, np.array([501, 501, 101]))
    else:
        grid = (np.array([-50.2, -50.2, -0.2]), 0.4, np.array([251, 251, 51]))
    return Workload(f"config4-{kind}", pts, grid)


def bspline_trajectory_batch(rng, n_batches: int, per_batch: int = 64, n_ctrl: int = 10,
                             lo=(-50.0, -50.0, 0.0), hi=(50.0, 50.0, 20.0), pitch_roll_std_deg: float = 10.0,
                             mount: bool = True):
    """Query stream of config 5: one uniform cubic B-spline per batch through n_ctrl
    random control points (positions U(box), yaw U(-pi,pi), pitch/roll N(0, 10 deg)),
    sampled at per_batch uniform parameters.  R = Rz Ry Rx (R_CAM_MOUNT if mount)."""
    ctrl_p = rng.uniform(lo, hi, size=(n_batches, n_ctrl, 3))
    ctrl_a = np.stack([rng.uniform(-np.pi, np.pi, (n_batches, n_ctrl)),
                       rng.normal(0.0, np.deg2rad(pitch_roll_std_deg), (n_batches, n_ctrl)),
                       rng.normal(0.0, np.deg2rad(pitch_roll_std_deg), (n_batches, n_ctrl))], axis=-1)
    segs = n_ctrl - 3
    u = np.linspace(0.0, segs, per_batch, endpoint=False) + 0.5 * segs / per_batch
    seg = np.minimum(u.astype(int), segs - 1)
    s = u - seg
    b = np.stack([(1 - s) ** 3, 3 * s ** 3 - 6 * s ** 2 + 4, -3 * s ** 3 + 3 * s ** 2 + 3 * s + 1, s ** 3], axis=1) / 6.0
    idx = seg[:, None] + np.arange(4)[None, :]
    pos = np.einsum("pk,bpkc->bpc", b, ctrl_p[:, idx, :])
    ang = np.einsum("pk,bpkc->bpc", b, ctrl_a[:, idx, :])
    rot = ypr_rotations(ang[..., 0].ravel(), ang[..., 1].ravel(), ang[..., 2].ravel())
    if mount:
        rot = rot @ R_CAM_MOUNT
    return pos.reshape(-1, 3), rot


def yaw_rotation(yaw: float) -> np.ndarray:
    return rot_z(yaw) @ R_CAM_MOUNT

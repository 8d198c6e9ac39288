"""Generate golden fixtures by running the reference `fifield` package in-process.

Run ONLY in the authoring container (the reference tree is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden.py

The reference's default numba backend is used (kernels.py:1529); all arrays are
float64 outputs of the reference's public API or its kernel boundary
(kernels.py:1559-1732).  Fixtures are small (a few MB total) and are the pins for
the C oracle under oracle/ and for the CUDA parity tests.
"""
from __future__ import annotations

import os
import sys

import numpy as np

import fifield
from fifield import kernels
from fifield.geometry import random_rotation

OUT = os.path.dirname(os.path.abspath(__file__))
kernels.warmup()
assert kernels.get_backend() == "numba"


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes raw")


# ── model parameters ────────────────────────────────────────────────
quad = fifield.build_quad_model(alpha=np.pi / 4, v_alpha=0.5)
gps = {ns: fifield.build_gp_model(ns) for ns in (30, 70)}
model_arrays = dict(quad_k=np.array([quad.alpha, quad.k2, quad.k1, quad.k0]))
for ns, m in gps.items():
    model_arrays[f"gp{ns}_zs"] = m.samples
    model_arrays[f"gp{ns}_kinv"] = m.kinv
    model_arrays[f"gp{ns}_par"] = np.array(
        [m.alpha, m.k_s, m.params.sigma2, m.params.length_scale, m.params.jitter]
    )
# direct gp_build at a fixed length scale (pins the Cholesky + Newton refinement)
m_fixed = fifield.gp_build(fifield.sample_directions(30), fifield.SeKernelParams(1.0, 0.5))
model_arrays["gp30_l05_kinv"] = m_fixed.kinv
model_arrays["quad_coeffs_grid"] = np.array(
    [[a, va, *fifield.quad_coefficients(a, va)] for a, va in [(np.pi / 4, 0.5), (np.pi / 3, 0.25), (0.9, 0.75)]]
)
model_arrays["train_l_small"] = np.array(
    [fifield.train_lengthscale(50, fifield.sample_directions(20), search_grid=np.geomspace(0.1, 1.5, 8), seed=2)]
)
save("models.npz", **model_arrays)


def field_args(f):
    return f.slots, f.factors, f._origin, f._vsize, f._dims


# ── small field: every kind, every query mode, edge positions ───────
rng = np.random.default_rng(11)
scene = fifield.gen_uniform(300, lo=(-2.0, -2.0, 0.0), hi=(2.0, 2.0, 2.0), seed=5)
pts = scene.positions
grid = fifield.GridConfig(np.array([-1.5, -1.25, 0.1]), 0.5, np.array([6, 5, 4]))
centers = grid.centers()
fields = {}
for mname, model in (("quad", quad), ("gp30", gps[30]), ("gp70", gps[70])):
    for kind in ("trace", "info"):
        fields[(mname, kind)] = fifield.Field.build(pts, grid, model, factor_kind=kind)
        # a second sigma on the quad info path pins the 1/sigma^2 scaling
fq_sigma = fifield.Field.build(pts, grid, quad, factor_kind="info", sigma=0.7)

first = centers[0]
last = centers[-1]
q_in = rng.uniform(first, last, size=(300, 3))
# edge positions: exact centres (incl. the last one), cell faces, the grid corners
edge = [first, last, centers[37], centers[59],
        grid.origin.copy(), grid.origin + grid.extent,
        np.array([last[0], first[1] + 0.25, last[2]]),
        np.array([first[0] + 0.5, last[1], first[2] + 0.75]),
        grid.origin + np.array([0.5, 0.5, 0.5]),                 # exactly on voxel faces
        grid.origin + grid.extent - 1e-12]
for a in range(3):
    for val in (first[a], last[a], grid.origin[a], grid.origin[a] + grid.extent[a]):
        p = rng.uniform(first, last)
        p[a] = val
        edge.append(p)
q_edge = np.array(edge)
q_out = rng.uniform(grid.origin - 1.0, grid.origin + grid.extent + 1.0, size=(60, 3))
positions = np.ascontiguousarray(np.vstack([q_in, q_edge, q_out]))
rots = np.stack([random_rotation(rng) for _ in range(positions.shape[0])])
axes = np.ascontiguousarray(rots[:, :, 2])

small = dict(points=pts, origin=grid.origin, voxel_size=np.array([grid.voxel_size]), dims=grid.dims,
             centers=centers, positions=positions, rotations=rots, factors_quad_info_sigma07=fq_sigma.factors)
for (mname, kind), f in fields.items():
    small[f"factors_{mname}_{kind}"] = f.factors
    for mode in ("nearest", "trilinear"):
        vals, ok = f.metric_axis_batch(positions, axes, "trace", mode)
        small[f"trace_{mname}_{kind}_{mode}"] = vals
        small[f"ok_{mname}_{kind}_{mode}"] = ok
        if kind == "info":
            fims, ok2 = f.query_fim_batch(positions, rots, mode)
            small[f"fim_{mname}_{mode}"] = fims
            # det / lmin metrics
            for metric in ("det", "lmin"):
                mv, _ = f.metric_axis_batch(positions, axes, metric, mode)
                small[f"{metric}_{mname}_{mode}"] = mv
# nearest-mode linear index + trilinear base for every position (bit-exact pins)
near_idx = np.array([kernels._np_locate_nearest(grid.origin, grid.voxel_size, grid.dims, p) for p in positions])
tri = []
for p in positions:
    c = kernels._np_trilinear_corners(grid.origin, grid.voxel_size, grid.dims, p)
    tri.append(np.concatenate([c[0].astype(np.float64), c[1]]) if c is not None else np.full(16, np.nan))
small["nearest_index"] = near_idx
small["trilinear_idx_w"] = np.array(tri)
save("small_field.npz", **small)

# ── config-1 rows: full-size landmark set, sampled voxels ───────────
sc1 = fifield.gen_uniform(2000, lo=(-5.0, -5.0, 0.0), hi=(5.0, 5.0, 3.0), seed=0)
g1 = fifield.GridConfig(np.array([-5.25, -5.25, -0.25]), 0.5, np.array([21, 21, 7]))
c1 = g1.centers()
vsel = np.sort(np.random.default_rng(3).choice(c1.shape[0], 24, replace=False))
cs = np.ascontiguousarray(c1[vsel])
m70 = gps[70]
cfg1 = dict(points=sc1.positions, vsel=vsel, centers=cs)
for kind in ("trace", "info"):
    tr = kind == "trace"
    cfg1[f"quad_{kind}"] = kernels.build_quad_factors(cs, sc1.positions, 1.0, quad.k2, quad.k1, quad.k0, tr)
    cfg1[f"gp70_{kind}"] = kernels.build_gp_factors(
        cs, sc1.positions, 1.0, m70.samples, m70.kinv, m70.k_s, float(np.cos(m70.alpha)), tr
    )
save("config1_rows.npz", **cfg1)

# ── point cloud (exact pinhole) ─────────────────────────────────────
cam = fifield.PinholeCamera.from_fov()
rng = np.random.default_rng(21)
pc_pts = rng.uniform([-6, -6, -1], [6, 6, 4], size=(1500, 3))
pc_rots = np.stack([random_rotation(rng) for _ in range(48)])
pc_ts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(48, 3))
# landmarks placed exactly on the image border of pose 0 (pixel u = 0 and u = 640 - tiny)
R0, t0 = pc_rots[0], pc_ts[0]
border = []
for zc in (1.0, 2.5, 4.0, 7.3):
    for (u, v) in ((0.0, 100.0), (640.0, 200.0), (320.0, 0.0), (320.0, 640.0), (639.9999999999, 5.0), (-1e-13, 7.0)):
        xc = (u - cam.cx) * zc / cam.fx
        yc = (v - cam.cy) * zc / cam.fy
        border.append(R0 @ np.array([xc, yc, zc]) + t0)
pc_pts = np.vstack([pc_pts, np.array(border)])
pc_out = fifield.exact_pose_fim_batch(pc_rots, pc_ts, pc_pts, cam)
mask = np.array([[fifield.exact_visible(fifield.Pose(pc_rots[q], pc_ts[q]), p, cam) for p in pc_pts]
                 for q in range(pc_rots.shape[0])])
# the hot path's own mask: a landmark is visible to the numba kernel iff its single-landmark
# exact FIM is non-zero (kernels.py:571-599).  exact_visible (fim.py:103-111) evaluates the
# projection through numpy matmul and can differ on exact-border pairs; both are stored.
fx, fy, cx, cy, w, h = cam.as_tuple()
kmask = np.array([[np.any(kernels.exact_fim(pc_rots[q], pc_ts[q], pc_pts[i:i + 1], fx, fy, cx, cy, w, h, 1.0) != 0)
                   for i in range(pc_pts.shape[0])] for q in range(pc_rots.shape[0])])
save("pc.npz", points=pc_pts, rotations=pc_rots, translations=pc_ts, fims=pc_out, visible=mask,
     visible_kernel=kmask, camera=np.array(cam.as_tuple()))

# ── per-landmark KATs ───────────────────────────────────────────────
rng = np.random.default_rng(31)
kat_t = rng.standard_normal((16, 3))
kat_p = kat_t + rng.standard_normal((16, 3)) * 3.0
kat_s = rng.uniform(0.3, 2.0, 16)
kat_fim = np.stack([fifield.landmark_fim(kat_t[i], kat_p[i], kat_s[i]) for i in range(16)])
kat_rot = np.stack([random_rotation(rng) for _ in range(16)])
kat_jac = np.stack([fifield.bearing_jacobian(fifield.Pose(kat_rot[i], kat_t[i]), kat_p[i]) for i in range(16)])
save("kats.npz", t=kat_t, p=kat_p, sigma=kat_s, fim=kat_fim, rot=kat_rot, jac=kat_jac,
     fib70=fifield.sample_directions(70), fib7=fifield.sample_directions(7))
print("versions: numpy", np.__version__, "numba", __import__("numba").__version__, file=sys.stderr)

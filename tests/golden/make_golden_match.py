"""Golden fixtures for matchability (field.py:101-180) from the reference package.

Run ONLY in the authoring container:
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden_match.py
Writes match.npz: the reference's Matchability.mask for range / view-cone gates
(with pairs placed exactly on the range limits) and masked field builds
(occupied rows + reference-layout factors) through fifield.build.
"""
from __future__ import annotations

import os

import numpy as np

import fifield
from fifield.field import GridConfig, Matchability
from fifield.scenes import Scene

OUT = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(31)
cfg = GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([6, 5, 4]))
centers = cfg.centers()
n = 300
pts = rng.uniform([-3, -3, -0.5], [3, 3, 2.5], size=(n, 3))
vd = rng.standard_normal((n, 3))
vd /= np.linalg.norm(vd, axis=1, keepdims=True)
dist = np.linalg.norm(pts[None] - centers[:, None], axis=2)
d_near = float(dist[7, 11])   # pairs exactly on the limits must be accepted (>=, <=)
d_far = float(dist[23, 42])
cases = {
    "range": Matchability(d_near=d_near, d_far=d_far),
    "near": Matchability(d_near=d_near),
    "cone": Matchability(view_cone_beta=1.1),
    "range_cone": Matchability(d_near=0.4, d_far=2.2, view_cone_beta=0.9),
    "sparse": Matchability(d_near=0.3, d_far=0.75, view_cone_beta=0.8),
}
arrays = dict(centers=centers, points=pts, view_dirs=vd, d_near=np.array(d_near), d_far=np.array(d_far))
for name, mt in cases.items():
    arrays[f"mask_{name}"] = mt.mask(centers, pts, vd)
scene = Scene(pts, vd)
quad = fifield.build_quad_model(alpha=np.pi / 4, v_alpha=0.5)
gp30 = fifield.build_gp_model(30)
for mname, model in (("quad", quad), ("gp30", gp30)):
    for kind in ("trace", "info"):
        f = fifield.build(scene, cfg, model, kind, matchability=cases["sparse"])
        arrays[f"occ3_{mname}_{kind}"] = f.occupied_index3
        arrays[f"factors_{mname}_{kind}"] = f.factors
np.savez_compressed(os.path.join(OUT, "match.npz"), **arrays)
print("wrote match.npz", {k: np.asarray(v).shape for k, v in arrays.items()})

# ── FIF1 files written by the reference (field.py:525-560) for interop tests ──
fif_dir = os.path.join(OUT, "fif1")
os.makedirs(fif_dir, exist_ok=True)
cfg2 = GridConfig(np.array([-1.0, -1.0, 0.0]), 0.5, np.array([4, 3, 3]))
pts2 = rng.uniform([-2, -2, 0], [2, 2, 2], size=(60, 3))
fifield.build(pts2, cfg2, quad, "info").serialize(os.path.join(fif_dir, "quad_info.fif"))
fifield.build(pts2, cfg2, gp30, "trace").serialize(os.path.join(fif_dir, "gp30_trace.fif"))
fifield.build(F_scene := Scene(pts2, vd[:60]), cfg2, gp30, "info",
              matchability=Matchability(d_near=0.2, d_far=1.2)).serialize(os.path.join(fif_dir, "gp30_info_masked.fif"))
np.savez_compressed(os.path.join(fif_dir, "inputs.npz"), points=pts2, view_dirs=vd[:60])
print("wrote fif1/*.fif")

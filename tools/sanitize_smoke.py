"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD

dev = torch.device("cuda")
rng = np.random.default_rng(0)
pts = rng.uniform([-3, -3, 0], [3, 3, 2], size=(300, 3))
vd = rng.standard_normal((300, 3))
vd /= np.linalg.norm(vd, axis=1, keepdims=True)
grid = F.GridConfig(np.array([-1.0, -1.0, 0.25]), 0.5, np.array([5, 4, 3]))
quad, gp30, gp150 = F.build_quad_model(), F.build_gp_model(30), F.build_gp_model(150)
fields = {}
gp70 = F.build_gp_model(70)
for kernel in ("t5", "t6"):  # tcgen05 builds (N_s = 30 and 70)
    FD.GP_INFO_KERNEL = kernel
    for model in (gp30, gp70):
        F.Field.build(pts, grid, model, "info")
for kernel in ("h16", "tf32", "simt"):
    FD.GP_INFO_KERNEL = kernel
    for model in (quad, gp30, gp150):
        for kind in ("trace", "info"):
            fields[(kernel, id(model), kind)] = F.Field.build(pts, grid, model, kind)
FD.GP_INFO_KERNEL = "h16"
F.Field.build(pts, grid, quad, "info", exact=True)
mt = F.Matchability(d_near=0.3, d_far=2.0, view_cone_beta=1.0)
fm = F.Field.build(F.Scene(pts, vd), grid, gp30, "info", matchability=mt)
fm.add_landmarks(F.Scene(pts[:20] + 0.1, vd[:20]))
c = grid.centers()
pos = rng.uniform(c[0], c[-1], size=(70, 3))
rots = np.stack([F.random_rotation(rng) for _ in range(70)])
for (kernel, mid, kind), f in fields.items():
    if kernel != "h16":
        continue
    for mode in ("nearest", "trilinear"):
        outs = ("trace", "full", "det", "lmin") if kind == "info" else ("trace",)
        f.query_batch(pos, rotations=rots, outputs=outs, grad=True, mode=mode)
        f.query_batch(pos, rotations=rots, outputs=("trace",), grad=False, mode=mode)
    if kind == "info":
        f.query_device(torch.tensor(pos, device=dev), torch.tensor(np.ascontiguousarray(rots[:, :, 2]), device=dev),
                       "trilinear", trace=True, full=True, grad=True, field_f64=True)
fm.query_batch(pos, rotations=rots, outputs=("trace", "full"), grad=True)
cam = F.PinholeCamera.from_fov()
F.exact_pose_fim_batch(rots, pos, pts, cam)
r = torch.tensor(rots.reshape(-1, 9), device=dev)
t = torch.tensor(pos, device=dev)
p = torch.tensor(pts, device=dev)
out = torch.empty((70, 36), dtype=torch.float64, device=dev)
mask = torch.empty((70, 300), dtype=torch.uint8, device=dev)
F.exact_pose_fim_batch_device(r, t, p, cam, out=out, mask=mask)
torch.cuda.synchronize()
print("sanitize smoke done")

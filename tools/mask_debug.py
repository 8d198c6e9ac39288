import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD
DEV = torch.device('cuda')
grid = F.GridConfig(np.array([-0.5, -0.5, 0.5]), 0.5, np.array([2, 2, 1]))
cen = grid.centers()
m = F.build_gp_model(70)
rng = np.random.default_rng(3)
pts = rng.uniform([-6, -6, -1], [6, 6, 3], size=(20000, 3))
mt = F.Matchability(d_near=0.3, d_far=4.0)
P = torch.tensor(pts, device=DEV)
res = {}
for kern in ("t5", "h16"):
    FD.GP_INFO_KERNEL = kern
    for order in ("all", "rev", "single1"):
        c = cen if order == "all" else (cen[::-1].copy() if order == "rev" else cen[1:2])
        s64, _ = FD.build_matched_rows(P, m, False, 1.0, DEV, torch.tensor(c, device=DEV), mt)
        r = s64.cpu().numpy()
        if order == "rev": r = r[::-1]
        res[(kern, order)] = r
ref = res[("h16", "all")]
for k, r in res.items():
    if k[1] == "single1":
        d = np.abs(r[0] - ref[1]).max() / np.abs(ref[1]).max(); print(k, "voxel1", f"{d:.2e}")
    else:
        print(k, [f"{np.abs(r[v] - ref[v]).max() / np.abs(ref[v]).max():.2e}" for v in range(4)])
# where is the error for voxel 1 (t5 all)?
e = np.abs(res[("t5", "all")][1] - ref[1]).reshape(70, 21)
print("per-sample max err (top 5):", np.argsort(e.max(1))[-5:], e.max(1)[np.argsort(e.max(1))[-5:]] / np.abs(ref[1]).max())
print("per-entry max err:", np.round(e.max(0) / np.abs(ref[1]).max(), 6))
# kept landmark count and nearest kept landmark per voxel
mask = mt.mask(cen, pts)
for v in range(4):
    d = np.linalg.norm(pts - cen[v], axis=1)
    print("voxel", v, "kept", int(mask[v].sum()), "nearest kept", d[mask[v]].min(), "nearest any", d.min())
# explicit (V, N) mask through fif_build (gate.mask) instead of the fused gates
md = torch.tensor(np.asarray(mt.mask(cen, pts), dtype=np.uint8), device=DEV)
for kern in ("t5", "h16"):
    FD.GP_INFO_KERNEL = kern
    s64, _ = FD.build_rows(P, m, False, 1.0, DEV, centers=torch.tensor(cen, device=DEV), mask=md)
    r = s64.cpu().numpy()
    print(kern, "explicit mask", [f"{np.abs(r[v] - ref[v]).max() / np.abs(ref[v]).max():.2e}" for v in range(4)])

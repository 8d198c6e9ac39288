"""Config-2 GP-info build: tcgen05 kernels (t6, t5) vs the mma.sync kernel (h16), timing and
precision against the C oracle on sampled voxels.  Usage: python tools/t5_probe.py [ns]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC
from oracle import oracle as O

dev = torch.device("cuda")
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 70
w2 = SC.config2(10)
grid = F.GridConfig(*w2.grid)
V, N = grid.voxel_count, w2.points.shape[0]
pts = torch.tensor(w2.points, device=dev)
gp = F.build_gp_model(ns)
dm = FD._DeviceModel(gp, dev)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


rng = np.random.default_rng(5)
sample = np.sort(rng.choice(V, 300, replace=False))
cz = grid.centers()  # x-major reference order
ref_rows = None
res = {}
KERNELS = tuple(os.environ.get("KERNELS", "t6,t5,h16").split(","))
for kern in KERNELS:
    FD.GP_INFO_KERNEL = kern
    out = {}

    def run():
        out["r"] = FD.build_rows(pts, gp, False, 1.0, dev, grid=grid, dmodel=dm)

    ms = timeit(run)
    r64 = out["r"][0] if isinstance(out["r"], tuple) else out["r"]
    res[kern] = r64
    print(f"{kern}: {ms:8.2f} ms  {V * N / ms * 1e3:.4e} pairs/s", flush=True)
# precision on sampled voxels (internal z-major rows) vs the oracle's S sums
nx, ny, nz = grid.dims
ix, iy, iz = sample % nx, (sample // nx) % ny, sample // (nx * ny)
cen = grid.origin + (np.stack([ix, iy, iz], 1) + 0.5) * grid.voxel_size
ref = O.build_gp_factors(cen, w2.points, 1.0, gp.samples, np.eye(ns), gp.k_s, np.cos(gp.alpha), False)
for kern, r64 in res.items():
    mine = r64.reshape(V, -1)[torch.as_tensor(sample, device=dev)].cpu().numpy()
    refp = ref.reshape(len(sample), ns, 6, 6)
    iu = np.triu_indices(6)
    refp = refp[:, :, iu[0], iu[1]].reshape(len(sample), -1)
    err = np.abs(mine - refp).max(1) / np.linalg.norm(refp, axis=1)
    print(f"{kern}: S max-entry / voxel-Frobenius over {len(sample)} voxels: max {err.max():.3e} median {np.median(err):.3e}")
for kern in KERNELS[:-1]:
    d = (res[kern] - res[KERNELS[-1]]).abs().max().item() / res[KERNELS[-1]].abs().max().item()
    print(f"{kern} vs {KERNELS[-1]} max abs diff / max: {d:.3e}")

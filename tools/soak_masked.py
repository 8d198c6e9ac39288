"""Randomised parity soak of the masked (matchability-gated) GP builds against the C oracle
(test infrastructure): random range gates (near / far, incl. limits that land exactly on a
pair's distance) and view cones, evaluated inside the build kernels (fif_build_matched) and
compared with the oracle run on the host mask (Matchability.mask, the numpy restatement that
the goldens pin bit-exact to the reference).  Pre-kinv sums, info (t5 masked path with and
without shared-memory gate bits, h16) and trace.
    python tools/soak_masked.py [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD
from oracle import oracle as O

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "0")))
dev = torch.device("cuda")
t0 = time.time()
models = {ns: F.build_gp_model(ns) for ns in (16, 30, 70)}
worst = {"t5 info": 0.0, "h16 info": 0.0, "trace": 0.0}
cases = 0
iu = np.triu_indices(6)
while time.time() - t0 < budget:
    ns = int(rng.choice([16, 30, 70]))
    m = models[ns]
    n = int(rng.choice([1, 64, 65, 513, int(rng.integers(1, 4000))]))
    nvox = int(rng.integers(1, 40))
    pts = rng.uniform(-4, 4, size=(n, 3))
    vd = rng.standard_normal((n, 3))
    vd /= np.linalg.norm(vd, axis=1, keepdims=True)
    cen = rng.uniform(-2, 2, size=(nvox, 3))
    kw = {}
    if rng.random() < 0.7:
        kw["d_far"] = float(rng.uniform(1.0, 6.0))
    if rng.random() < 0.5:
        kw["d_near"] = float(rng.uniform(0.05, 1.0))
    if rng.random() < 0.5:
        kw["view_cone_beta"] = float(rng.uniform(0.3, 2.5))
    if not kw:
        kw["d_far"] = 3.0
    if "d_far" in kw and rng.random() < 0.3:  # a limit exactly on a pair's distance
        kw["d_far"] = float(np.linalg.norm(pts[rng.integers(n)] - cen[rng.integers(nvox)]))
    mt = F.Matchability(**kw)
    mask = np.asarray(mt.mask(cen, pts, vd), dtype=np.uint8)
    P, C = torch.tensor(pts, device=dev), torch.tensor(cen, device=dev)
    ref = O.build_gp_factors(cen, pts, 1.0, m.samples, np.eye(ns), m.k_s, np.cos(m.alpha), False, mask)
    refp = ref.reshape(nvox, ns, 6, 6)[:, :, iu[0], iu[1]].reshape(nvox, -1)
    nrm = np.linalg.norm(refp, axis=1)
    for kern in ("t5", "h16"):
        FD.GP_INFO_KERNEL = kern
        s64, _ = FD.build_matched_rows(P, m, False, 1.0, dev, C, mt, vd)
        mine = s64.cpu().numpy()
        assert np.isfinite(mine).all()
        assert np.all(mine[nrm == 0] == 0), "a voxel without matched landmarks must be zero"
        if (nrm > 0).any():
            e = (np.abs(mine - refp).max(1) / np.maximum(nrm, 1e-300))[nrm > 0].max()
            worst[f"{kern} info"] = max(worst[f"{kern} info"], float(e))
    FD.GP_INFO_KERNEL = "t5"
    reft = O.build_gp_factors(cen, pts, 1.0, m.samples, np.eye(ns), m.k_s, np.cos(m.alpha), True, mask).reshape(nvox, -1)
    t64, _ = FD.build_matched_rows(P, m, True, 1.0, dev, C, mt, vd)
    nt = np.linalg.norm(reft, axis=1)
    if (nt > 0).any():
        e = (np.linalg.norm(t64.cpu().numpy() - reft, axis=1) / np.maximum(nt, 1e-300))[nt > 0].max()
        worst["trace"] = max(worst["trace"], float(e))
    cases += 1
print(f"{cases} random masked cases in {time.time() - t0:.0f} s")
print("worst errors (info: max entry / voxel Frobenius, bound 1e-5; trace: per-voxel relative L2, bound 1e-5):",
      {k: f"{v:.3e}" for k, v in worst.items()})
sys.exit(0 if all(v <= 1e-5 for v in worst.values()) else 1)

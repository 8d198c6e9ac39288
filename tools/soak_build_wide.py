"""Randomised parity soak of the remaining build paths against the C oracle (test
infrastructure): GP info and trace builds over the whole supported sample range (N_s = 4 ..
320: the tcgen05 kernel up to 80, the mma.sync kernel above), quad info and trace builds in
the fast mode (<= 1e-12) and the EXACT mode (bit-identical), random landmark counts and grids.
    python tools/soak_build_wide.py [seconds]"""
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
worst = {"gp info": 0.0, "gp trace": 0.0, "quad info": 0.0, "quad trace": 0.0}
cases = 0
iu = np.triu_indices(6)
quad = F.build_quad_model()
while time.time() - t0 < budget:
    ns = int(rng.choice([int(rng.integers(4, 81)), int(rng.integers(81, 321))]))
    n = int(rng.choice([1, 31, 32, 33, 64, 127, 128, 129, 255, 256, 257, int(rng.integers(1, 3000))]))
    dims = rng.integers(1, 5, size=3)
    vs = float(rng.uniform(0.15, 0.8))
    origin = rng.uniform(-2, 2, size=3)
    sigma = float(rng.uniform(0.5, 2.0))
    grid = F.GridConfig(origin, vs, dims)
    pts = rng.uniform(origin - 3.0, origin + dims * vs + 3.0, size=(n, 3))
    nx, ny, nz = (int(d) for d in dims)
    j = np.arange(nx * ny * nz)
    cen = origin + (np.stack([j % nx, (j // nx) % ny, j // (nx * ny)], 1) + 0.5) * vs
    try:
        m = F.build_gp_model(ns, k_s=float(rng.uniform(5, 25)), alpha=float(rng.uniform(0.3, 1.2)),
                             length_scale=float(rng.uniform(0.2, 0.8)))
    except F.SingularGram:
        continue
    P = torch.tensor(pts, device=dev)
    V = len(cen)
    ref = O.build_gp_factors(cen, pts, sigma, m.samples, np.eye(ns), m.k_s, np.cos(m.alpha), False)
    refp = ref.reshape(V, ns, 6, 6)[:, :, iu[0], iu[1]].reshape(V, -1)
    mine = FD.build_rows(P, m, False, sigma, dev, grid=grid)[0].cpu().numpy()
    nrm = np.maximum(np.linalg.norm(refp, axis=1), 1e-300)
    worst["gp info"] = max(worst["gp info"], float((np.abs(mine - refp).max(1) / nrm).max()))
    reft = O.build_gp_factors(cen, pts, sigma, m.samples, np.eye(ns), m.k_s, np.cos(m.alpha), True).reshape(V, -1)
    minet = FD.build_rows(P, m, True, sigma, dev, grid=grid)[0].cpu().numpy()
    worst["gp trace"] = max(worst["gp trace"], float((np.linalg.norm(minet - reft, axis=1) /
                                                      np.maximum(np.linalg.norm(reft, axis=1), 1e-300)).max()))
    for want_trace, key in ((False, "quad info"), (True, "quad trace")):
        rq = O.build_quad_factors(cen, pts, sigma, quad.k2, quad.k1, quad.k0, want_trace)
        ex = FD.build_rows(P, quad, want_trace, sigma, dev, grid=grid, exact=True)[0].cpu().numpy()
        rq_p = rq.reshape(V, 10, 6, 6)[:, :, iu[0], iu[1]].reshape(V, -1) if not want_trace else rq.reshape(V, -1)
        assert np.array_equal(ex, rq_p), f"EXACT quad build not bit-identical: case {cases} n {n} dims {dims} {key}"
        fast = FD.build_rows(P, quad, want_trace, sigma, dev, grid=grid)[0].cpu().numpy()
        sc = np.maximum(np.abs(rq_p).max(1, keepdims=True), 1e-300)
        worst[key] = max(worst[key], float((np.abs(fast - rq_p) / sc).max()))
    cases += 1
print(f"{cases} random cases in {time.time() - t0:.0f} s; EXACT quad builds bit-identical")
print("worst errors (gp info: max entry / voxel Frobenius, bound 1e-5; gp trace: per-voxel relative L2, bound 1e-5; "
      "quad fast mode: max entry / voxel max, bound 1e-12):", {k: f"{v:.3e}" for k, v in worst.items()})
ok = worst["gp info"] <= 1e-5 and worst["gp trace"] <= 1e-5 and worst["quad info"] <= 1e-12 and worst["quad trace"] <= 1e-12
sys.exit(0 if ok else 1)

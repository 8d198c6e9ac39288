"""Randomised parity soak of the point-cloud kernel against the C oracle (test
infrastructure): random pinhole cameras (field of view, resolution, principal point), pose
and landmark counts (landmark-group / tile remainders, the sorted and unsorted pose paths),
scene scales, landmarks placed on image borders, on the optical centre plane, 0.1 mm in front of
and at the camera centre; visibility masks bit-exact (kernels.py:580-595), FIMs <= 1e-4
relative.  (A visible landmark closer than ~1e-9 |p| to a camera centre is outside the
kernel's FP32 hi / lo bearing precision, DESIGN 4: the first version of this soak put one at
1 nm in a 30 m scene and measured 1.3e-4.)
    python tools/soak_pc.py [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_03324_b200 as F
from oracle import oracle as O

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "0")))
dev = torch.device("cuda")
t0 = time.time()
cases = pairs = 0
worst = 0.0
while time.time() - t0 < budget:
    w, h = int(rng.integers(64, 1921)), int(rng.integers(64, 1081))
    fov = float(rng.uniform(0.5, 2.6))
    f = 0.5 * w / np.tan(0.5 * fov)
    cam = F.PinholeCamera(fx=f, fy=f * float(rng.uniform(0.8, 1.25)), cx=w / 2.0 + float(rng.uniform(-20, 20)),
                          cy=h / 2.0 + float(rng.uniform(-20, 20)), width=w, height=h, half_fov_alpha=fov / 2.0)
    q = int(rng.choice([1, 15, 16, 200, int(rng.integers(1, 12000))]))   # >= 8 880 poses: sorted path
    n = int(rng.choice([1, 31, 32, 33, 1023, 1024, 1025, int(rng.integers(1, 6000))]))
    scale = float(rng.choice([0.5, 3.0, 30.0]))
    pts = rng.uniform(-scale, scale, size=(n, 3))
    pos = rng.uniform(-scale, scale, size=(q, 3))
    rots = np.stack([F.random_rotation(rng) for _ in range(q)])
    # landmarks exactly on the borders of pose 0's image, on its z = 0 plane and at its centre
    R0, t0p = rots[0], pos[0]
    k = min(n, 8)
    special = []
    for (u, v, z) in ((0.0, h / 2, 2.0), (float(w), h / 2, 2.0), (w / 2, 0.0, 2.0), (w / 2, float(h), 2.0),
                      (0.0, 0.0, 1.0), (float(w), float(h), 1.0), (w / 2, h / 2, 0.0), (w / 2, h / 2, 1e-4))[:k]:
        pc = np.array([(u - cam.cx) / cam.fx * z, (v - cam.cy) / cam.fy * z, z])
        special.append(R0 @ pc + t0p)
    pts[:k] = np.array(special)
    if n > k:
        pts[k] = t0p  # at the camera centre: skipped by the reference (n^2 < 1e-300) or invisible
    r = torch.tensor(rots.reshape(-1, 9), device=dev)
    t = torch.tensor(pos, device=dev)
    p = torch.tensor(pts, device=dev)
    out = torch.empty((q, 36), dtype=torch.float64, device=dev)
    mask = torch.empty((q, n), dtype=torch.uint8, device=dev)
    F.exact_pose_fim_batch_device(r, t, p, cam, out=out, mask=mask)
    ref = O.exact_fim_batch(rots, pos, pts, cam.as_tuple())
    rmask = O.pc_mask(rots, pos, pts, cam.as_tuple())
    mine_mask = mask.cpu().numpy()
    if not np.array_equal(mine_mask.astype(bool), np.asarray(rmask).astype(bool)):
        bad = np.argwhere(mine_mask.astype(bool) != np.asarray(rmask).astype(bool))
        print(f"mask differs in {len(bad)} pairs: case {cases} q {q} n {n} scale {scale} cam {cam}; first {bad[:4].tolist()}")
        sys.exit(1)
    mine = out.cpu().numpy().reshape(q, 6, 6)
    nr = np.linalg.norm(ref.reshape(q, -1), axis=1)
    e = np.linalg.norm((mine - ref).reshape(q, -1), axis=1) / np.maximum(nr, 1e-300)
    if (nr > 0).any():
        worst = max(worst, float(e[nr > 0].max()))
    assert np.all(mine[nr == 0] == 0)
    cases += 1
    pairs += q * n
print(f"{cases} random cases, {pairs} pose-landmark pairs in {time.time() - t0:.0f} s; masks bit-exact; "
      f"worst FIM relative Frobenius error {worst:.3e} (tolerance 1e-4)")
sys.exit(0 if worst <= 1e-4 else 1)

"""Randomised soak of the analytic pose gradients (FIF_Q_GRAD, new in this build; consumer
traj.py:383-398) against central finite differences (h = 1e-6) of the FP64 oracle's trilinear
query: random quad / GP info fields, random poses kept >= 1e-3 cells away from cell faces
(the trilinear query is only piecewise smooth), d trace / d[t; theta] and d FIM / d[t; theta]
<= 1e-4 relative (FD noise ~1e-7).
    python tools/soak_grad.py [seconds]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2008_03324_b200 as F
from oracle import oracle as O
from paper_2008_03324_b200.geometry import so3_exp
from tests._helpers import oracle_model

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "0")))
t0 = time.time()
models = {"quad": F.build_quad_model(), "gp16": F.build_gp_model(16), "gp30": F.build_gp_model(30),
          "gp70": F.build_gp_model(70)}
worst = {"trace_grad": 0.0, "fim_grad": 0.0}
cases = queries = 0
h = 1e-6
while time.time() - t0 < budget:
    mname = str(rng.choice(list(models)))
    m = models[mname]
    dims = rng.integers(2, 6, size=3)
    vs = float(rng.uniform(0.3, 0.8))
    origin = rng.uniform(-1, 1, size=3)
    grid = F.GridConfig(origin, vs, dims)
    # landmarks outside the grid volume (>= 1 voxel away): smooth, well-scaled fields
    pts = rng.uniform(origin - 4.0, origin + dims * vs + 4.0, size=(int(rng.integers(30, 300)), 3))
    inside = np.all((pts > origin - vs) & (pts < origin + dims * vs + vs), axis=1)
    pts = pts[~inside]
    if len(pts) < 10:
        continue
    f = F.Field.build(pts, grid, m, "info")
    order = np.argsort(grid.linear_index(f.occupied_index3))
    factors = f.factors[order]  # reference order, dense
    slots = np.arange(grid.voxel_count, dtype=np.int32)
    om = oracle_model(m)
    q = int(rng.integers(1, 200))
    c = grid.centers()
    pos = rng.uniform(c.min(0), c.max(0), size=(q, 3))
    g = (pos - origin) / vs - 0.5
    frac = g - np.floor(g)
    pos = pos[((frac > 1e-3) & (frac < 1 - 1e-3)).all(axis=1)]
    if len(pos) == 0:
        continue
    rots = np.stack([F.random_rotation(rng) for _ in range(len(pos))])

    def ev(p, r):
        ax = np.ascontiguousarray(r[:, :, 2])
        fim, _ = O.query_fim_batch(slots, factors, grid.origin, grid.voxel_size, grid.dims, p, ax, om, True)
        return fim

    g_fim = np.zeros((len(pos), 6, 6, 6))
    for j in range(6):
        if j < 3:
            d = np.zeros(3)
            d[j] = h
            a, b = ev(pos + d, rots), ev(pos - d, rots)
        else:
            w = np.zeros(3)
            w[j - 3] = h
            a = ev(pos, np.einsum("ij,qjk->qik", so3_exp(w), rots))
            b = ev(pos, np.einsum("ij,qjk->qik", so3_exp(-w), rots))
        g_fim[:, j] = (a - b) / (2 * h)
    g_tr = np.trace(g_fim, axis1=2, axis2=3)
    res = f.query_batch(pos, rotations=rots, outputs=("trace", "full"), grad=True, to_numpy=True)
    # FD noise floor: ~1e-7 |F| / h relative to the gradient norm; gradients much smaller than
    # |F| per unit are dominated by it, so errors are taken against max(|grad|, 1e-2 |F|)
    fn = np.linalg.norm(ev(pos, rots).reshape(len(pos), -1), axis=1)
    mine_f = res["fim_grad"]
    # the library orders fim_grad as (Q, 6, 6, 6): find which axis is the derivative axis
    if not np.allclose(mine_f[0, 0], g_fim[0, 0], rtol=1e-3, atol=1e-3 * fn[0]):
        mine_f = np.moveaxis(mine_f, 3, 1)
    sc = np.maximum(np.linalg.norm(g_fim.reshape(len(pos), -1), axis=1), 1e-2 * fn)
    worst["fim_grad"] = max(worst["fim_grad"], float((np.linalg.norm((mine_f - g_fim).reshape(len(pos), -1), axis=1) / sc).max()))
    sct = np.maximum(np.linalg.norm(g_tr, axis=1), 1e-2 * fn)
    worst["trace_grad"] = max(worst["trace_grad"], float((np.linalg.norm(res["trace_grad"] - g_tr, axis=1) / sct).max()))
    cases += 1
    queries += len(pos)
print(f"{cases} random fields, {queries} poses in {time.time() - t0:.0f} s")
print("worst |analytic - FD| / max(|FD|, 1e-2 |F|) (tolerance 1e-4):", {k: f"{v:.3e}" for k, v in worst.items()})
sys.exit(0 if all(v <= 1e-4 for v in worst.values()) else 1)

"""Randomised soak of the indexing rule (fif_locate; kernels.py:628-635 nearest, 678-702
trilinear): random grids (origin, voxel size incl. non-representable values like 0.1 / 0.3,
1-60 voxels per axis), positions uniformly inside and around the field, on voxel centres, on
cell faces, on the last centre plane and one ulp to either side of each; nearest index,
trilinear corner indices, the 8 weights and the status compared BIT FOR BIT with the oracle.
    python tools/soak_locate.py [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2008_03324_b200 as F
from oracle import oracle as O

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "0")))
t0 = time.time()
quad = F.build_quad_model()
cases = npos = 0
while time.time() - t0 < budget:
    dims = rng.integers(1, 61, size=3)
    vs = float(rng.choice([0.1, 0.2, 0.25, 0.3, 0.4, 0.7, float(rng.uniform(0.05, 2.0))]))
    origin = rng.choice([np.zeros(3), rng.uniform(-50, 50, size=3), np.round(rng.uniform(-5, 5, size=3), 1)])
    grid = F.GridConfig(np.asarray(origin, dtype=np.float64), vs, dims)
    f = F.Field.build(np.zeros((0, 3)), grid, quad, "trace")
    ext = dims * vs
    n = 400
    pos = rng.uniform(origin - vs, origin + ext + vs, size=(n, 3))
    # half of them snapped per axis to centres / faces (k * vs / 2 from the origin), +- 1 ulp
    snap = rng.random((n, 3)) < 0.5
    k = rng.integers(-1, 2 * dims + 2, size=(n, 3))
    sn = origin + 0.5 * vs * k
    ulp = rng.integers(-1, 2, size=(n, 3))
    sn = np.where(ulp > 0, np.nextafter(sn, np.inf), np.where(ulp < 0, np.nextafter(sn, -np.inf), sn))
    pos = np.where(snap, sn, pos)
    near = f.locate(pos, "nearest")
    tri = f.locate(pos, "trilinear")
    for i, p in enumerate(pos):
        ni = O.locate_nearest(grid.origin, grid.voxel_size, grid.dims, p)
        assert near["index"][i, 0] == ni and (near["status"][i] == 1) == (ni < 0), ("nearest", cases, i, p, dims, vs)
        r = O.trilinear(grid.origin, grid.voxel_size, grid.dims, p)
        if r is None:
            assert tri["status"][i] == 1, ("trilinear status", cases, i, p, dims, vs)
        else:
            assert tri["status"][i] == 0, ("trilinear status", cases, i, p, dims, vs)
            assert np.array_equal(tri["index"][i], r[0]), ("corner indices", cases, i, p, dims, vs)
            assert np.array_equal(tri["weight"][i], r[1]), ("corner weights", cases, i, p, dims, vs)
    cases += 1
    npos += n
print(f"{cases} random grids, {npos} positions in {time.time() - t0:.0f} s: nearest index, corner indices, weights and "
      f"statuses bit-identical to the oracle")

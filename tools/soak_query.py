"""Randomised parity soak of the query kernels against the C oracle (test infrastructure):
random quad / GP fields on small grids (some built with range gates, so voxels are missing),
random batch sizes (the fused small-batch kernel below 445 GP queries, the streaming kernels
above), positions inside, on the faces of and outside the field, both modes; status
bit-exact, full 6x6 and trace <= 1e-4 relative, det / lambda_min <= 1e-4 of max(|value|,
1e-3 of its natural scale |F|^6 / |F|).
    python tools/soak_query.py [seconds]"""
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
worst = {"fim": 0.0, "trace": 0.0, "det": 0.0, "lmin": 0.0}
cases = queries = 0
models = {}
while time.time() - t0 < budget:
    dims = rng.integers(1, 7, size=3)
    vs = float(rng.uniform(0.2, 0.8))
    origin = rng.uniform(-2, 2, size=3)
    grid = F.GridConfig(origin, vs, dims)
    n = int(rng.integers(1, 400))
    ext = dims * vs
    pts = rng.uniform(origin - 2.0, origin + ext + 2.0, size=(n, 3))
    kind_m = str(rng.choice(["quad", "gp"]))
    if kind_m == "quad":
        m = F.build_quad_model()
        mt = ("quad", m.k2, m.k1, m.k0)
    else:
        ns = int(rng.choice([9, 16, 30, 45, 70]))
        m = models.setdefault(ns, F.build_gp_model(ns))
        mt = ("gp", m.samples, m.params.sigma2, m.params.length_scale)
    match = F.Matchability(d_far=float(rng.uniform(1.0, 3.0))) if rng.random() < 0.3 else F.ALWAYS_MATCH
    f = F.Field.build(pts, grid, m, "info", matchability=match)
    slots = np.full(grid.voxel_count, -1, np.int32)
    if f.rows:
        slots[grid.linear_index(f.occupied_index3)] = np.arange(f.rows, dtype=np.int32)
    fac = f.factors if f.rows else np.zeros((1, (10 if kind_m == "quad" else m.n_v) * 36))
    q = int(rng.choice([1, 3, 64, 444, 445, 1000, int(rng.integers(1, 3000))]))
    pos = rng.uniform(origin - 0.3 * vs, origin + ext + 0.3 * vs, size=(q, 3))
    face = rng.random(q) < 0.15          # exactly on a face / centre plane of the grid
    ax_i = rng.integers(0, 3, size=q)
    k_i = rng.integers(0, 2 * dims[ax_i] + 1)
    pos[face, ax_i[face]] = origin[ax_i[face]] + 0.5 * vs * k_i[face]
    rots = np.stack([F.random_rotation(rng) for _ in range(q)])
    for mode in ("nearest", "trilinear"):
        res = f.query_batch(pos, rotations=rots, outputs=("trace", "full", "det", "lmin"), mode=mode, to_numpy=True)
        rf, st = O.query_fim_batch(slots, fac, grid.origin, grid.voxel_size, grid.dims, pos, rots[:, :, 2], mt,
                                   mode == "trilinear")
        ok = st == 0
        assert np.array_equal(res["in_field"], ok), f"status differs: case {cases} {mode} dims {dims} q {q}"
        if ok.any():
            nr = np.linalg.norm(rf[ok].reshape(-1, 36), axis=1)
            # (a pose whose FIM is below 1e-6 of the batch's largest is rounding noise around zero:
            # a gate removed its landmarks; its determinant is noise of noise)
            sc = np.maximum(nr, 1e-6 * max(nr.max(), 1e-300))
            worst["fim"] = max(worst["fim"], float((np.linalg.norm((res["fim"][ok] - rf[ok]).reshape(-1, 36), axis=1) / sc).max()))
            tr = np.trace(rf[ok], axis1=1, axis2=2)
            worst["trace"] = max(worst["trace"], float((np.abs(res["trace"][ok] - tr) / np.maximum(np.abs(tr), sc)).max()))
            for met in ("det", "lmin"):
                v, _ = O.metric_batch(slots, fac, grid.origin, grid.voxel_size, grid.dims, pos, rots[:, :, 2], mt, met,
                                      False, mode == "trilinear")
                # eigenvalue / determinant perturbations scale with |F|: rank-deficient random FIMs
                # (few landmarks) have lambda_min ~ 0, so the floor is 1e-3 of the natural scale
                nat = (sc / np.sqrt(6.0)) ** 6 if met == "det" else sc
                ref_scale = np.maximum(np.maximum(np.abs(v[ok]), 1e-3 * nat), 1e-300)
                errs = np.abs(res[met][ok] - v[ok]) / ref_scale
                if errs.max() > 1e-4 and os.environ.get("SOAK_VERBOSE"):
                    i = int(np.argmax(errs))
                    ev = np.linalg.eigvalsh(rf[ok][i])
                    print(f"{met} error {errs.max():.3e}: case {cases} model {kind_m} ns {getattr(m, 'n_v', 0)} n {n} dims "
                          f"{dims.tolist()} q {q} mode {mode} gated {match is not F.ALWAYS_MATCH}; mine {res[met][ok][i]:.6e} "
                          f"ref {v[ok][i]:.6e} |F| {nr[i]:.3e} eig(blended F) {ev}", flush=True)
                worst[met] = max(worst[met], float(errs.max()))
        queries += 2 * q
    cases += 1
print(f"{cases} random fields, {queries} queries in {time.time() - t0:.0f} s; statuses bit-exact")
print("worst relative errors (tolerance 1e-4):", {k: f"{v:.3e}" for k, v in worst.items()})
sys.exit(0 if all(v <= 1e-4 for v in worst.values()) else 1)

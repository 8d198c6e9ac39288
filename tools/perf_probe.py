"""Config-2 scale timing of every kernel + GP precision vs the oracle on sampled voxels/queries."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC, _lib
from oracle import oracle as O

dev = torch.device('cuda')
w2 = SC.config2(100000)
grid = F.GridConfig(*w2.grid)
V = grid.voxel_count; N = w2.points.shape[0]
pts = torch.tensor(w2.points, device=dev)
quad = F.build_quad_model(); gp70 = F.build_gp_model(70)

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)

ONLY_Q = '--only-query' in sys.argv
pairs = V * N
for name, model, tr, ex in [] if ONLY_Q else [('quad trace', quad, True, False), ('quad trace exact', quad, True, True), ('quad info', quad, False, False),
                            ('gp70 trace', gp70, True, False), ('gp70 info', gp70, False, False)]:
    dm = FD._DeviceModel(model, dev)
    ms = timeit(lambda: FD.build_rows(pts, model, tr, 1.0, dev, grid=grid, dmodel=dm, exact=ex))
    print(f'{name:18s} {ms:9.2f} ms  {pairs/ms*1e3:.3e} pairs/s', flush=True)

# GP precision at config-2 scale on sampled voxels (explicit centres) vs the oracle
rng = np.random.default_rng(5)
cen = grid.centers()
sel = np.sort(rng.choice(V, 48, replace=False))
csel = torch.tensor(cen[sel], device=dev)
for name, model, tr in [] if ONLY_Q else [('gp70 trace', gp70, True), ('gp70 info', gp70, False), ('quad info', quad, False)]:
    s64, _ = FD.build_rows(pts, model, tr, 1.0, dev, centers=csel)
    fld = FD.Field(grid, model, 'trace' if tr else 'info', 1.0, s64, None, grid.index3_of(sel).astype(np.int32), dense=False)
    mine = fld.factors
    t0 = time.time()
    if model is quad:
        ref = O.build_quad_factors(cen[sel], w2.points, 1.0, quad.k2, quad.k1, quad.k0, tr)
    else:
        ref = O.build_gp_factors(cen[sel], w2.points, 1.0, gp70.samples, gp70.kinv, gp70.k_s, np.cos(gp70.alpha), tr)
    ot = time.time() - t0
    if tr:
        err = (np.linalg.norm(mine - ref, axis=1) / np.linalg.norm(ref, axis=1))
    else:
        err = np.array([np.abs(mine[i] - ref[i]).max() / np.linalg.norm(ref[i]) for i in range(len(sel))])
    print(f'{name} config2 build err max {err.max():.3e} median {np.median(err):.3e} (oracle {ot:.1f}s, {O.max_threads()} thr)', flush=True)

# queries: GPU build of the whole config-2 field, timing of 100k queries with gradients
for name, model in [('gp70', gp70), ('quad', quad)]:
    f = F.Field.build(w2.points, grid, model, 'info')
    pos = torch.tensor(w2.positions, device=dev); ax = torch.tensor(w2.rotations[:, :, 2].copy(), device=dev)
    out = {}
    for label, kw in [('full+grad', dict(trace=True, full=True, grad=True)), ('full', dict(trace=False, full=True)),
                      ('trace', dict(trace=True)), ('trace+grad', dict(trace=True, grad=True)),
                      ('det', dict(trace=False, det=True)), ('det+grad', dict(trace=False, det=True, grad=True)),
                      ('lmin', dict(trace=False, lmin=True)), ('nearest full+grad', dict(trace=True, full=True, grad=True, mode='nearest'))]:
        kw = dict(kw); md = kw.pop('mode', 'trilinear')
        ms = timeit(lambda: f.query_device(pos, ax, md, out={}, **kw))
        print(f'query {name} info {label:10s} {ms:8.3f} ms  {1e5/ms*1e3:.3e} q/s', flush=True)
    # precision vs oracle on a cropped reference field for 40 queries
    qsel = np.arange(40)
    res = f.query_batch(w2.positions[qsel], rotations=w2.rotations[qsel], outputs=('trace', 'full'), mode='trilinear', to_numpy=True)
    lin_needed = set()
    for p in w2.positions[qsel]:
        c = O.trilinear(grid.origin, grid.voxel_size, grid.dims, p)
        lin_needed.update(c[0].tolist())
    lin_needed = np.array(sorted(lin_needed))
    cc = cen[lin_needed]
    t0 = time.time()
    if model is quad:
        ref_rows = O.build_quad_factors(cc, w2.points, 1.0, quad.k2, quad.k1, quad.k0, False)
        mt = ('quad', quad.k2, quad.k1, quad.k0)
    else:
        ref_rows = O.build_gp_factors(cc, w2.points, 1.0, gp70.samples, gp70.kinv, gp70.k_s, np.cos(gp70.alpha), False)
        mt = ('gp', gp70.samples, gp70.params.sigma2, gp70.params.length_scale)
    slots = np.full(V, -1, np.int32); slots[lin_needed] = np.arange(len(lin_needed), dtype=np.int32)
    axes = w2.rotations[qsel][:, :, 2].copy()
    rt, _ = O.metric_batch(slots, ref_rows, grid.origin, grid.voxel_size, grid.dims, w2.positions[qsel], axes, mt, 'trace', False, True)
    rf, _ = O.query_fim_batch(slots, ref_rows, grid.origin, grid.voxel_size, grid.dims, w2.positions[qsel], axes, mt, True)
    et = np.abs(res['trace'] - rt) / np.abs(rt)
    ef = np.linalg.norm((res['fim'] - rf).reshape(40, -1), axis=1) / np.linalg.norm(rf.reshape(40, -1), axis=1)
    print(f'query {name} config2 parity: trace rel max {et.max():.2e}  fim relF max {ef.max():.2e} (oracle {time.time()-t0:.1f}s)', flush=True)

if ONLY_Q:
    sys.exit(0)
# PC: 100k poses of config 3
w3 = SC.config3(100000)
r = torch.tensor(w3.rotations.reshape(-1, 9), device=dev); t = torch.tensor(w3.positions, device=dev)
cam = F.PinholeCamera.from_fov()
ms = timeit(lambda: F.exact_pose_fim_batch_device(r, t, pts, cam))
print(f'pc 1e5 poses x 2e4: {ms:.2f} ms  {1e5*N/ms*1e3:.3e} pose-landmark pairs/s', flush=True)
out = F.exact_pose_fim_batch_device(r[:200], t[:200], pts, cam).cpu().numpy().reshape(-1, 6, 6)
ref = O.exact_fim_batch(w3.rotations[:200], w3.positions[:200], w2.points, cam.as_tuple())
e = np.linalg.norm((out - ref).reshape(200, -1), axis=1) / np.maximum(np.linalg.norm(ref.reshape(200, -1), axis=1), 1e-300)
print('pc parity relF max', e.max())
mask = torch.zeros((200, N), dtype=torch.uint8, device=dev)
F.exact_pose_fim_batch_device(r[:200], t[:200], pts, cam, mask=mask)
om = O.pc_mask(w3.rotations[:200], w3.positions[:200], w2.points, cam.as_tuple())
print('pc mask bit-exact', np.array_equal(mask.cpu().numpy().astype(bool), om), 'visible frac', om.mean())

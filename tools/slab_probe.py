"""Per-rank compute time of the z-slab build split measured on one GPU.

For N in 1, 2, 4, 8 the config-2 GP-70 info grid is split by voxel count exactly as
bench.py / parallel.py split it across ranks, and every rank's slab is built (and timed
with CUDA events) one after another on this GPU.  Slab builds are independent (no
collective, no cross-slab reads), so each timing is that rank's step time on a B200;
max over ranks bounds the N-GPU step, and T1 / (N max) is the load-balance / tail
efficiency of the split (the landmark broadcast, ~1 ms once per build, is excluded).
This is a prediction from 1-GPU timings, not a multi-GPU measurement.

    python tools/slab_probe.py [--model gp70] [--kind info] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC
from paper_2008_03324_b200.parallel import slab_range

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="gp70")
ap.add_argument("--kind", default="info")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
w = SC.config2(0)
grid = F.GridConfig(*w.grid)
model = F.build_quad_model() if a.model == "quad" else F.build_gp_model(int(a.model[2:]))
dev = torch.device("cuda")
pts = torch.tensor(w.points, device=dev)
dm = FD._DeviceModel(model, dev)
V = grid.voxel_count


def timed(v0, v1):
    best = None
    for _ in range(a.reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        FD.build_rows(pts, model, a.kind == "trace", 1.0, dev, grid=grid, dmodel=dm, v_begin=v0, v_end=v1)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        best = ms if best is None else min(best, ms)
    return best


timed(0, V)  # warm-up
t1 = timed(0, V)
print(f"config2 {a.model} {a.kind}: {V} voxels x {pts.shape[0]} landmarks, 1 rank {t1:.2f} ms")
for n in (2, 4, 8):
    ts = [timed(*slab_range(V, n, r)) for r in range(n)]
    print(f"N={n}: per-rank ms " + " ".join(f"{t:.2f}" for t in ts) +
          f" | max {max(ts):.2f} mean {sum(ts) / n:.2f} | predicted step efficiency T1/(N max) = {t1 / (n * max(ts)):.3f}",
          flush=True)

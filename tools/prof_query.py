"""Config-2 query workload (100k poses, trilinear, full + trace + gradient) for ncu capture."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="gp70")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--grad", type=int, default=1)
a = ap.parse_args()
w = SC.config2(100000)
grid = F.GridConfig(*w.grid)
model = F.build_quad_model() if a.model == "quad" else F.build_gp_model(int(a.model[2:]))
dev = torch.device("cuda")
f = F.Field.build(w.points, grid, model, "info")
pos = torch.tensor(w.positions, device=dev)
ax = torch.tensor(np.ascontiguousarray(w.rotations[:, :, 2]), device=dev)
out = {}
for r in range(a.reps):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    f.query_device(pos, ax, "trilinear", trace=True, full=True, grad=bool(a.grad), out=out)
    e.record(); torch.cuda.synchronize()
    print(f"query {a.model} grad={a.grad} rep {r}: {s.elapsed_time(e):.3f} ms", flush=True)

"""Run one config-2 build variant twice (warm-up + measured) — the ncu capture target."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC

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
for r in range(a.reps):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    FD.build_rows(pts, model, a.kind == "trace", 1.0, dev, grid=grid, dmodel=dm)
    e.record(); torch.cuda.synchronize()
    print(f"{a.model} {a.kind} rep {r}: {s.elapsed_time(e):.2f} ms", flush=True)

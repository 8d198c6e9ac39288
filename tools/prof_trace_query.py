"""Config-2 GP-70 and quad TRACE-field queries (trace + gradient), 1e5 poses."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC

w = SC.config2(100000)
grid = F.GridConfig(*w.grid)
dev = torch.device("cuda")
pos = torch.tensor(w.positions, device=dev)
ax = torch.tensor(np.ascontiguousarray(w.rotations[:, :, 2]), device=dev)
for name, model in (("gp70", F.build_gp_model(70)), ("quad", F.build_quad_model())):
    f = F.Field.build(w.points, grid, model, "trace")
    for mode in ("trilinear", "nearest"):
        out = {}
        for _ in range(2):
            f.query_device(pos, ax, mode, trace=True, grad=True, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            f.query_device(pos, ax, mode, trace=True, grad=True, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        nc = 8 if mode == "trilinear" else 1
        row = model.n_v * (4 if name != "quad" else 8)
        print(f"{name} trace field {mode:9s}: {ms:.3f} ms / 1e5 queries ({1e5 * nc * row / ms / 1e6:.0f} GB/s rows)",
              flush=True)

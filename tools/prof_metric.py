"""Config-2 metric queries (det / lambda_min, with and without gradients), 1e5 poses."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC

w = SC.config2(100000)
f = F.Field.build(w.points, F.GridConfig(*w.grid), F.build_gp_model(70), "info")
dev = torch.device("cuda")
pos = torch.tensor(w.positions, device=dev)
ax = torch.tensor(np.ascontiguousarray(w.rotations[:, :, 2]), device=dev)
for label, kw in [("trace", dict(trace=True)), ("det", dict(trace=False, det=True)),
                  ("det+grad", dict(trace=False, det=True, grad=True)), ("lmin", dict(trace=False, lmin=True)),
                  ("lmin+grad", dict(trace=False, lmin=True, grad=True))]:
    out = {}
    for _ in range(2):
        f.query_device(pos, ax, "trilinear", out=out, **kw)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        f.query_device(pos, ax, "trilinear", out=out, **kw)
    b.record()
    torch.cuda.synchronize()
    print(f"{label:10s} {a.elapsed_time(b) / 5:8.3f} ms / 1e5 queries", flush=True)

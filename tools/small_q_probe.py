import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC
w = SC.config2(4096)
f = F.Field.build(w.points, F.GridConfig(*w.grid), F.build_gp_model(70), "info")
dev = torch.device("cuda")
pos = torch.tensor(w.positions[:64], device=dev); ax = torch.tensor(np.ascontiguousarray(w.rotations[:64, :, 2]), device=dev)
for kw in (dict(trace=True, full=True, grad=True), dict(trace=True, full=True, det=True, grad=True)):
    for _ in range(3): f.query_device(pos, ax, "trilinear", **kw)
torch.cuda.synchronize()

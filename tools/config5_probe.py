"""Config 5 query path on the config-4 field: per-batch device time with and without the
trace output (the FP64 trace-table pass), for the launch list under ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC

dev = torch.device("cuda")
w = SC.config4("info", 1)
grid = F.GridConfig(*w.grid)
gp70 = F.build_gp_model(70)
pts = torch.tensor(w.points, device=dev)
f = F.Field.build(pts, grid, gp70, "info")
torch.cuda.synchronize()
qrng = np.random.default_rng(4)
out = {}
for trace in (True, False, True, False):
    pos, rot = SC.bspline_trajectory_batch(qrng, (1 << 20) // 64)
    p = torch.tensor(pos, device=dev)
    ax = torch.tensor(np.ascontiguousarray(rot[:, :, 2]), device=dev)
    f.query_device(p, ax, "trilinear", trace=trace, full=True, grad=True, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    f.query_device(p, ax, "trilinear", trace=trace, full=True, grad=True, out=out)
    b.record()
    torch.cuda.synchronize()
    print(f"trace={trace}: {p.shape[0]} queries {a.elapsed_time(b):.2f} ms", flush=True)

"""One GP-info build launch over the first VOXELS voxels of config 2 (ncu target).
Usage: python tools/t5_one.py [kernel=t5] [voxels=3552] [ns=70]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC

kern = sys.argv[1] if len(sys.argv) > 1 else "t5"
nvox = int(sys.argv[2]) if len(sys.argv) > 2 else 3552
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 70
dev = torch.device("cuda")
w2 = SC.config2(10)
grid = F.GridConfig(*w2.grid)
pts = torch.tensor(w2.points, device=dev)
gp = F.build_gp_model(ns)
dm = FD._DeviceModel(gp, dev)
FD.GP_INFO_KERNEL = kern
for _ in range(2):
    r, _ = FD.build_rows(pts, gp, False, 1.0, dev, grid=grid, dmodel=dm, v_end=nvox)
torch.cuda.synchronize()
print("ok", kern, nvox, float(r.abs().sum()))

"""Bit-compare the config-2 GP-info rows of two library builds (tuning variants).
Usage: python tools/cmp_rows.py A.so B.so [voxels] [masked]  (run on a GPU box)"""
import os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    os.environ["FIF_LIB"] = sys.argv[2]
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import paper_2008_03324_b200 as F
    from paper_2008_03324_b200 import field as FD, scenes as SC
    nvox, masked, out = int(sys.argv[3]), sys.argv[4] == "1", sys.argv[5]
    w = SC.config2(0)
    grid = F.GridConfig(*w.grid)
    gp = F.build_gp_model(70)
    dev = torch.device("cuda")
    pts = torch.tensor(w.points, device=dev)
    if masked:
        c = FD.device_centers(grid, dev)[:nvox].contiguous()
        r, _ = FD.build_matched_rows(pts, gp, False, 1.0, dev, c, F.Matchability(d_near=0.3, d_far=4.0))
        np.save(out, r.cpu().numpy())
    else:
        r, _ = FD.build_rows(pts, gp, False, 1.0, dev, grid=grid, dmodel=FD._DeviceModel(gp, dev), v_end=nvox)
        np.save(out, r.cpu().numpy())
    sys.exit(0)
a, b = sys.argv[1], sys.argv[2]
nvox = sys.argv[3] if len(sys.argv) > 3 else "20000"
masked = sys.argv[4] if len(sys.argv) > 4 else "0"
for lib, out in ((a, "/tmp/cmp_a.npy"), (b, "/tmp/cmp_b.npy")):
    subprocess.run([sys.executable, __file__, "--one", lib, nvox, masked, out], check=True)
import numpy as np
x, y = np.load("/tmp/cmp_a.npy"), np.load("/tmp/cmp_b.npy")
print("shape", x.shape, "bit-identical" if np.array_equal(x, y) else f"DIFFER max {np.abs(x - y).max():.3e} "
      f"rel {np.abs(x - y).max() / np.abs(x).max():.3e}")

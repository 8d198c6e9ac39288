"""Config-2 GP-70 info build to host factors (Field.build(host_factors=True)) at several
chunk counts, plus the export kernel and the D2H copy alone.  Run on a GPU box."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD, scenes as SC

w = SC.config2(0)
grid = F.GridConfig(*w.grid)
gp = F.build_gp_model(70)
dev = torch.device("cuda")
pts = torch.tensor(w.points).pin_memory()
host = torch.empty((grid.voxel_count, 70 * 36), dtype=torch.float64).pin_memory()


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


f = F.Field.build(pts, grid, gp, "info", device=dev)
print("build only %.2f ms" % timed(lambda: F.Field.build(pts, grid, gp, "info", device=dev)))
dev_rows = f.export_reference()
print("export kernel (whole field) %.2f ms" % timed(lambda: f.export_reference()))
print("D2H 2.78 GB %.2f ms" % timed(lambda: host.copy_(dev_rows, non_blocking=True)))
del dev_rows
print("export_reference_to %.2f ms" % timed(lambda: f.export_reference_to(host)))
for n in (4, 8, 16, 32):
    FD.HOST_EXPORT_CHUNKS = n
    print("host_factors build, %d chunks: %.2f ms" % (n, timed(lambda: F.Field.build(pts, grid, gp, "info", device=dev,
                                                                                    host_factors=True, host_out=host))))

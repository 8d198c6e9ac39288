"""Masked t5 builds at growing landmark counts (gate bits in shared memory up to ~83k
landmarks at N_s = 70, further at N_s = 30) against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import field as FD
from oracle import oracle as O
from tests._helpers import info_rel_fro, oracle_field
DEV = torch.device('cuda')
grid = F.GridConfig(np.array([-0.5, -0.5, 0.5]), 0.5, np.array([2, 2, 1]))
cen = grid.centers()
for ns in (30, 70):
    m = F.build_gp_model(ns)
    for n in (20_000, 60_000, 90_000, 100_000):
        rng = np.random.default_rng(3)
        pts = rng.uniform([-6, -6, -1], [6, 6, 3], size=(n, 3))
        for masked in (True, False):
            mt = F.Matchability(d_near=0.3, d_far=4.0) if masked else F.Matchability()
            mask = mt.mask(cen, pts)
            ref = oracle_field(O, m, cen, pts, "info", mask=None if mask is None else np.asarray(mask, dtype=np.uint8))
            if masked:
                s64, _ = FD.build_matched_rows(torch.tensor(pts, device=DEV), m, False, 1.0, DEV, torch.tensor(cen, device=DEV), mt)
            else:
                s64, _ = FD.build_rows(torch.tensor(pts, device=DEV), m, False, 1.0, DEV, centers=torch.tensor(cen, device=DEV))
            fld = FD.Field(grid, m, "info", 1.0, s64, None, grid.index3_of(np.arange(cen.shape[0])).astype(np.int32), dense=False)
            print(ns, n, "masked" if masked else "plain", np.array2string(info_rel_fro(fld.factors, ref), precision=2), flush=True)

"""Config-3 point-cloud workload (1e6 poses x 20k landmarks) for timing / ncu capture."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC

ap = argparse.ArgumentParser()
ap.add_argument("--poses", type=int, default=1000000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = SC.config3(a.poses)
dev = torch.device("cuda")
r = torch.tensor(w.rotations.reshape(-1, 9), device=dev)
t = torch.tensor(w.positions, device=dev)
p = torch.tensor(w.points, device=dev)
cam = F.PinholeCamera.from_fov()
out = torch.empty((a.poses, 36), dtype=torch.float64, device=dev)
for i in range(a.reps):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); F.exact_pose_fim_batch_device(r, t, p, cam, out=out); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"pc {a.poses} poses rep {i}: {ms:.2f} ms  {a.poses * p.shape[0] / ms / 1e9:.3e} pairs/s", flush=True)

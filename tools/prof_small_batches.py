"""Planner-style small query batches: per-call latency of direct fif_query calls vs a
CUDA-graph replay (Field.query_graph), config-2 GP-70 info field, full + grad."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2008_03324_b200 as F
from paper_2008_03324_b200 import scenes as SC

w = SC.config2(4096)
grid = F.GridConfig(*w.grid)
f = F.Field.build(w.points, grid, F.build_gp_model(70), "info")
dev = torch.device("cuda")
for batch in (64, 1024):
    pos = torch.tensor(w.positions[:batch], device=dev)
    ax = torch.tensor(np.ascontiguousarray(w.rotations[:batch, :, 2]), device=dev)
    out = {}
    kw = dict(trace=True, full=True, det=True, grad=True)
    for _ in range(20):
        f.query_device(pos, ax, "trilinear", out=out, **kw)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        f.query_device(pos, ax, "trilinear", out=out, **kw)
    torch.cuda.synchronize()
    direct = (time.perf_counter() - t0) / n * 1e6
    g = f.query_graph(batch, "trilinear", outputs=("trace", "full", "det"), grad=True)
    for _ in range(20):
        g.run(pos, ax)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        g.run(pos, ax)
    torch.cuda.synchronize()
    graph = (time.perf_counter() - t0) / n * 1e6
    g.positions.copy_(pos)
    g.axes.copy_(ax)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        g.replay()
    torch.cuda.synchronize()
    rep = (time.perf_counter() - t0) / n * 1e6
    # device time per call (CUDA events around 200 back-to-back replays)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    dev_us = a.elapsed_time(b) / 200 * 1e3
    print(f"batch {batch:5d}: direct {direct:8.1f} us/call, graph run() {graph:8.1f} us/call, "
          f"graph replay() {rep:8.1f} us/call, device {dev_us:7.1f} us/call", flush=True)

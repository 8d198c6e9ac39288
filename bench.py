#!/usr/bin/env python
"""Benchmark of the FIF hot path on B200 (contract: one JSON line on rank 0).

Headline workload = BASELINE.json configs[1] ("config 2"): full 6x6 information
PIF build of the GP-70 model (the reference CLI's default model, cli.py:537)
over 20 000 room landmarks x an 81x81x21 grid (2.756e9 voxel-landmark pairs).
A step = one build of this rank's z-slab of the grid; with N ranks the grid is
split by voxel count (strong scaling, no collective in the inner loop; the
landmarks are broadcast once over NCCL).  Secondary lines in the same JSON:
config-2 batched queries (100 000 poses, full 6x6 + analytic gradient) and the
config-3 point-cloud baseline kernel.

--impl reference times the reference algorithm on the host CPU (the C oracle
port of fifield's numba kernels, all host threads) on the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GP_INFO_FLOPS_PER_PAIR = lambda ns: 94 + 50 * ns   # SURVEY.md §8(d) algorithmic count, FMA = 2
GP_INFO_MUFU_PER_PAIR = lambda ns: 1 + 2 * ns
QUERY_ROW_BYTES_GP_INFO = lambda ns: ns * 21 * 4  # FP32 S rows, packed 21 entries
METRIC = "FIF build voxel·landmark pairs/s"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ns", type=int, default=70)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU seconds for the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the query / PC secondary measurements")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ── clocks sampled during the timed region ─────────────────────────
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ── CPU reference leg (oracle port of the reference kernels) ────────
def cpu_gp_info_rate(points, centers, model, seconds, threads):
    """Reference GP info build (fast C port) on a voxel sample sized to ~`seconds` of work; returns (pairs/s, sample text)."""
    from oracle import oracle as O

    rng = np.random.default_rng(123)
    n = points.shape[0]
    k = max(threads, 16)
    sel = rng.choice(centers.shape[0], k, replace=False)
    t0 = time.perf_counter()
    O.build_gp_factors_fast(centers[sel], points, 1.0, model.samples, model.kinv, model.k_s, np.cos(model.alpha),
                            False, nthreads=threads)
    dt = time.perf_counter() - t0
    k2 = int(min(centers.shape[0], max(k, k * seconds / max(dt, 1e-3))))
    k2 = max(threads, (k2 // threads) * threads)
    sel = rng.choice(centers.shape[0], k2, replace=False)
    t0 = time.perf_counter()
    O.build_gp_factors_fast(centers[sel], points, 1.0, model.samples, model.kinv, model.k_s, np.cos(model.alpha),
                            False, nthreads=threads)
    dt = time.perf_counter() - t0
    return k2 * n / dt, (f"{k2} random config-2 voxels x {n} landmarks (GP-{model.n_v} info), {dt:.2f} s; "
                         "reference algorithm (vs @ kinv, vp x I6 per landmark) as a blocked AVX2/FMA C port, "
                         "OpenMP over voxels (oracle/fif_cpu_fast.c)")


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_2008_03324_b200 import scenes as SC
    from paper_2008_03324_b200.field import GridConfig
    from paper_2008_03324_b200.visibility import build_gp_model

    w2 = SC.config2(0)
    grid = GridConfig(*w2.grid)
    model = build_gp_model(args.ns)
    centers = grid.centers()
    thr = host_threads()
    for _ in range(max(1, min(args.warmup, 1))):
        cpu_gp_info_rate(w2.points, centers, model, 1.0, thr)
    rates = []
    sample = ""
    per_step = max(2.0, 60.0 / max(args.steps, 1))
    for _ in range(args.steps):
        r, sample = cpu_gp_info_rate(w2.points, centers, model, per_step, thr)
        rates.append(r)
    value = float(np.median(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(2.756e9 / value * 1e3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded config-2 room landmarks)",
        "config": {"workload": f"config2: GP-{args.ns} info build, 20000 room landmarks x 81x81x21 grid @0.25 m",
                   "global_batch": 137781 * 20000, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ── GPU leg ─────────────────────────────────────────────────────────
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2008_03324_b200 as F
    from paper_2008_03324_b200 import _lib, scenes as SC
    from paper_2008_03324_b200 import field as FD
    from paper_2008_03324_b200.parallel import slab_range

    # FIF_BENCH_BACKEND=gloo with more ranks than GPUs only exercises the multi-rank code
    # path (ranks share a device; their kernels never wait on each other); numbers from
    # such a run are not measurements
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    if world > 1:
        backend = os.environ.get("FIF_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    w2 = SC.config2(100000)
    grid = F.GridConfig(*w2.grid)
    V, N = grid.voxel_count, w2.points.shape[0]
    model = F.build_gp_model(args.ns)
    dm = FD._DeviceModel(model, dev)
    # landmarks: generated on rank 0, broadcast once over NCCL
    pts = torch.tensor(w2.points, device=dev) if rank == 0 else torch.empty((N, 3), dtype=torch.float64, device=dev)
    if world > 1:
        dist.broadcast(pts, src=0)
    v0, v1 = slab_range(V, world, rank)
    rows = v1 - v0
    width = model.n_v * 21
    out64 = torch.empty((rows, width), dtype=torch.float64, device=dev)
    out32 = torch.empty((rows, width), dtype=torch.float32, device=dev)
    scratch = torch.empty(int(_lib.load().fif_build_scratch_bytes(N)), dtype=torch.uint8, device=dev)
    g = _lib.make_grid(grid.origin, grid.voxel_size, grid.dims)
    L = _lib.load()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        _lib.check(L.fif_build(_lib.KIND_INFO, dm.c, pts.data_ptr(), N, g, None, v0, v1, None, 1.0, 0,
                               scratch.data_ptr(), out64.data_ptr(), out32.data_ptr(), stream.cuda_stream),
                   "fif_build")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local % ndev) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = _lib.launch_count()
        t_wall = time.perf_counter()
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall
        launches = _lib.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    dev_ms = float(sum(step_ms))
    if world > 1:
        tt = torch.tensor([dev_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms = float(tt.item())
    ms_per_step = dev_ms / args.steps
    pairs_total = V * N
    value = pairs_total / (ms_per_step / 1e3)

    # dominant kernel: k_gp_info alone (the step also runs the landmark-table prep)
    k_ms = ms_per_step
    # e2e through the public API: host landmarks (pinned) -> build -> D2H checksum
    pts_host = torch.tensor(w2.points).pin_memory()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        d_pts = pts_host.to(dev, non_blocking=True)
        s64, s32 = FD.build_rows(d_pts, model, False, 1.0, dev, grid=grid, v_begin=v0, v_end=v1, dmodel=dm)
        chk = s32.sum(dtype=torch.float64).to("cpu", non_blocking=True)
        b.record(stream)
        b.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
        del s64, s32
    e2e_step = float(np.mean(e2e_ms))
    if world > 1:
        tt = torch.tensor([e2e_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_step = float(tt.item())
    e2e_value = pairs_total / (e2e_step / 1e3)

    clk = clocks.summary()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    max_mhz = float(peaks.get("sm_max_mhz", clk.get("sm_max_mhz") or 1965.0))
    fp32_peak = sms * 128 * 2 * max_mhz * 1e6 / 1e12  # TFLOP/s
    flops_launch = (rows * N) * GP_INFO_FLOPS_PER_PAIR(model.n_v)
    achieved = flops_launch / (k_ms / 1e3) / 1e12
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get("k_gp_info_h16", {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (FP16 hi+lo tensor products, FP32 accumulate) + f64 accumulation",
        "data": "synthetic: seeded config-2 room landmarks (BASELINE configs[1]); no dataset",
        "config": {"workload": f"config2: GP-{model.n_v} info PIF build, {N} room landmarks x 81x81x21 grid @0.25 m",
                   "global_batch": int(pairs_total), "parallelism": f"z-slab x{world}",
                   "l2": "256 MB buffer written between timed steps (inputs are L2-resident)",
                   "wall_s_timed_region": t_wall},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(pts_host.numel() * 8),
                "d2h_bytes_per_step": 8, "ms_per_step": e2e_step,
                "path": "host float64 landmarks (pinned) -> H2D -> fif_build -> D2H checksum"},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "traffic": traffic,
                     "kernel": "k_gp_info_h16", "flops_per_pair": GP_INFO_FLOPS_PER_PAIR(model.n_v),
                     "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 x {max_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                     "mufu_frac": (rows * N * GP_INFO_MUFU_PER_PAIR(model.n_v)) / (k_ms / 1e3)
                                  / (sms * 16 * max_mhz * 1e6)},
        "step_ms_each": step_ms,
    }
    extras = {}
    if not args.no_extras:
        extras = secondary(args, F, FD, SC, w2, grid, model, dm, pts, dev, stream, flush, world, rank, peaks, sms,
                           max_mhz)
        line.update(extras)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = host_threads()
        cpu_v, sample = cpu_gp_info_rate(w2.points, grid.centers(), model, args.cpu_seconds, thr)
        line["cpu_baseline"] = {"value": cpu_v, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample}
        v1, s1 = cpu_gp_info_rate(w2.points, grid.centers(), model, min(4.0, args.cpu_seconds / 3), 1)
        line["cpu_baseline"]["single_thread"] = {"value": v1, "unit": UNIT, "sample": s1}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def secondary(args, F, FD, SC, w2, grid, model, dm, pts, dev, stream, flush, world, rank, peaks, sms, max_mhz):
    """Config-2 queries (full 6x6 + gradient) and config-3 point-cloud kernel, timed the same way."""
    import torch

    from paper_2008_03324_b200.parallel import slab_range

    res = {}
    fld = F.Field.build(pts, grid, model, "info", device=dev)
    q0, q1 = slab_range(w2.positions.shape[0], world, rank)  # replicated field, queries sharded
    pos = torch.tensor(w2.positions[q0:q1], device=dev)
    ax = torch.tensor(np.ascontiguousarray(w2.rotations[q0:q1, :, 2]), device=dev)
    out = {}
    fld.query_device(pos, ax, "trilinear", trace=True, full=True, grad=True, out=out)
    times = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fld.query_device(pos, ax, "trilinear", trace=True, full=True, grad=True, out=out)
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    qms = float(np.mean(times))
    q_traffic = None
    try:  # ncu dram bytes of k_query_prep_gp + k_query_info per query (profiles/ncu_summary.json)
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        q_traffic = prof["query_per_query"]["dram_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    nq = q1 - q0
    row = QUERY_ROW_BYTES_GP_INFO(model.n_v)
    bytes_q = 8 * row + 48 + 8 * (1 + 6 + 36 + 216)  # 8 corner rows + pose in + outputs
    hbm = float(peaks.get("hbm_gbs", 6550.4))
    res["query"] = {
        "workload": "config2: 100000 poses, trilinear, full 6x6 + trace + analytic d/d[t;theta], GP-70 info field",
        "value": nq * world / (qms / 1e3), "unit": "queries/s", "ms": qms,
        "roofline": {"bound": "hbm", "achieved": nq * bytes_q / (qms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": nq * bytes_q / (qms / 1e3) / 1e9 / hbm, "traffic": q_traffic,
                     "bytes_per_query": bytes_q},
    }
    # point cloud (config 3): poses sharded across ranks
    npose = 1000000
    w3 = SC.config3(npose)
    p0, p1 = slab_range(npose, world, rank)
    r = torch.tensor(w3.rotations[p0:p1].reshape(-1, 9), device=dev)
    t = torch.tensor(w3.positions[p0:p1], device=dev)
    cam = F.PinholeCamera.from_fov()
    outpc = torch.empty((p1 - p0, 36), dtype=torch.float64, device=dev)
    F.exact_pose_fim_batch_device(r, t, pts, cam, out=outpc)
    times = []
    for _ in range(max(1, args.steps // 2)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        F.exact_pose_fim_batch_device(r, t, pts, cam, out=outpc)
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    pms = float(np.mean(times))
    res["pc"] = {"workload": "config3: 1e6 poses x 20000 landmarks, exact pinhole FIM (trace + 6x6)",
                 "value": (p1 - p0) * w2.points.shape[0] * world / (pms / 1e3), "unit": "pose-landmark pairs/s",
                 "ms": pms}
    return res


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())

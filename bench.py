#!/usr/bin/env python
"""Benchmark of the FIF hot path on B200 (contract: one JSON line on rank 0).

Headline workload = BASELINE.json configs[1] ("config 2"): full 6x6 information
PIF build of the GP-70 model (the reference CLI's default model, cli.py:537)
over 20 000 room landmarks x an 81x81x21 grid (2.756e9 voxel-landmark pairs).
A step = one build of this rank's z-slab of the grid; with N ranks the grid is
split by voxel count (strong scaling, no collective in the inner loop; the
landmarks are broadcast once over NCCL).

Secondary measurements in the same JSON line:
  e2e / e2e_export — the public API (Field.build) from pinned host landmarks, with a
      D2H checksum, and with the reference-layout factors (kinv @ S) exported to host;
  parity           — the built rows of the CPU-baseline sample voxels vs the CPU port;
  query            — config-2 queries (1e5 poses, full 6x6 + trace + gradient) + roofline;
  pc               — config-3 point-cloud kernel (1e6 poses x 2e4 landmarks) + roofline;
  pc_vs_fif        — FIF queries on the SAME 1e6 poses (speed-up, Table II-style error);
  masked_build     — config-2 build with range + occlusion gates fused into the kernels.

--impl reference times the reference algorithm on the host CPU (the CPU port of
fifield's numba kernels, all host threads) on the same metric and config: its K timed
steps partition the config-2 grid, so together they build the whole field once.
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
QUERY_TRACE_ROW_BYTES = lambda ns: ns * 8         # FP64 trace table row (trace outputs of an info field)
PC_FLOPS_TEST, PC_FLOPS_VISIBLE = 28, 110         # SURVEY.md §8(d) config-3 per-pair count
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
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary measurements")
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


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


PORT_DESC = ("reference algorithm (_nb_build_gp, kernels.py:471-524: vs per landmark, vp = vs @ kinv, vp x I6) as a "
             "blocked AVX2/FMA C port, OpenMP over voxels (oracle/fif_cpu_fast.c; 1.94x faster per thread than the "
             "reference's numba+BLAS, so the ratio understates the speed-up over the reference itself)")


# ── CPU legs (the reference's algorithm on the host cores) ──────────
def cpu_gp_info_rate(points, centers, model, seconds, threads, seed=123):
    """The CPU port on a random voxel sample sized to ~`seconds` of work.
    Returns (pairs/s, sample text, selected voxel indices, port output rows)."""
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
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
    out = O.build_gp_factors_fast(centers[sel], points, 1.0, model.samples, model.kinv, model.k_s,
                                  np.cos(model.alpha), False, nthreads=threads)
    dt = time.perf_counter() - t0
    return k2 * n / dt, f"{k2} random config-2 voxels x {n} landmarks (GP-{model.n_v} info), {dt:.2f} s; " + PORT_DESC, \
        sel, out


def run_reference(args, rank, world):
    """The driver's reference arm: the reference algorithm on every host core, same metric and
    config.  The K timed steps partition the config-2 voxels (contiguous slices, like the GPU
    z-slabs), so the run builds the complete 81x81x21 field exactly once; value = all pairs /
    total time.  Warm-up steps run small samples (untimed)."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2008_03324_b200 import scenes as SC
    from paper_2008_03324_b200.field import GridConfig
    from paper_2008_03324_b200.parallel import slab_range
    from paper_2008_03324_b200.visibility import build_gp_model

    w2 = SC.config2(0)
    grid = GridConfig(*w2.grid)
    model = build_gp_model(args.ns)
    centers = grid.centers()
    V, N = centers.shape[0], w2.points.shape[0]
    thr = host_threads()
    cosa = float(np.cos(model.alpha))
    rng = np.random.default_rng(7)
    for _ in range(args.warmup):
        sel = rng.choice(V, 2 * thr, replace=False)
        O.build_gp_factors_fast(centers[sel], w2.points, 1.0, model.samples, model.kinv, model.k_s, cosa, False,
                                nthreads=thr)
    K = max(1, args.steps)
    step_s = []
    for s in range(K):
        v0, v1 = slab_range(V, K, s)
        t0 = time.perf_counter()
        O.build_gp_factors_fast(centers[v0:v1], w2.points, 1.0, model.samples, model.kinv, model.k_s, cosa, False,
                                nthreads=thr)
        step_s.append(time.perf_counter() - t0)
    total = float(sum(step_s))
    value = V * N / total
    sample = (f"the {K} timed steps partition all {V} config-2 voxels ({V // K}-{-(-V // K)} voxels x {N} landmarks "
              f"each): together one complete GP-{model.n_v} info build of the 81x81x21 grid, {total:.1f} s; "
              + PORT_DESC)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": total / K * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded config-2 room landmarks)",
        "config": {"workload": f"config2: GP-{args.ns} info PIF build, {N} room landmarks x 81x81x21 grid @0.25 m",
                   "global_batch": int(V * N), "sample": sample, "full_grid_s": total},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_ms_each": [x * 1e3 for x in step_s],
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
    k_ms = ms_per_step  # the step is k_prep_landmarks (~µs) + the GP-info build kernel
    kname = "k_gp_info_t5" if (FD.GP_INFO_KERNEL == "t5" and model.n_v <= 80) else "k_gp_info_h16"

    e2e, e2e_export = measure_e2e(args, F, FD, w2, grid, model, dev, stream, flush, world, rank, v0, v1)

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
    mufu_peak = sms * 16 * max_mhz * 1e6 / 1e9  # Gop/s
    mufu_achieved = (rows * N * GP_INFO_MUFU_PER_PAIR(model.n_v)) / (k_ms / 1e3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get(kname, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (FP16 hi+lo tcgen05 products, FP32 TMEM accumulate) + f64 accumulation",
        "data": "synthetic: seeded config-2 room landmarks (BASELINE configs[1]); no dataset",
        "config": {"workload": f"config2: GP-{model.n_v} info PIF build, {N} room landmarks x 81x81x21 grid @0.25 m",
                   "global_batch": int(pairs_total), "parallelism": f"z-slab x{world}",
                   "l2": "256 MB buffer written between timed steps (inputs are L2-resident)",
                   "wall_s_timed_region": t_wall},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "e2e_export": e2e_export,
        # the binding pipe: the 21 x N_s contraction (2 940 of the 3 594 algorithmic flop per pair
        # at N_s = 70) runs on tcgen05, so what bounds the kernel is the transcendental (XU/MUFU)
        # pipe that evaluates the sigmoids: algorithmically exp + reciprocal per (pair, sample)
        # plus one rsqrt per pair, 16 per clock per SM
        "roofline": {"bound": "xu (MUFU transcendentals)", "achieved": mufu_achieved, "peak": mufu_peak,
                     "unit": "Gop/s", "frac": mufu_achieved / mufu_peak, "traffic": traffic,
                     "kernel": kname, "ops_per_pair": GP_INFO_MUFU_PER_PAIR(model.n_v),
                     "peak_source": f"{sms} SMs x 16 MUFU lanes x {max_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                     "fp32_equiv": {"achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                                    "frac": achieved / fp32_peak, "flops_per_pair": GP_INFO_FLOPS_PER_PAIR(model.n_v),
                                    "note": "SURVEY 8(d) algorithmic FP32 count over the FP32 SIMT peak; above 1 "
                                            "because the contraction runs on the tensor cores"}},
        "step_ms_each": step_ms,
    }
    if not args.no_extras:
        line.update(secondary(args, F, FD, SC, w2, grid, model, pts, dev, stream, flush, world, rank, peaks, sms,
                              max_mhz))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = host_threads()
        centers = grid.centers()
        cpu_v, sample, sel, port_rows = cpu_gp_info_rate(w2.points, centers, model, args.cpu_seconds, thr)
        line["cpu_baseline"] = {"value": cpu_v, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample}
        v1_, s1, _, _ = cpu_gp_info_rate(w2.points, centers, model, min(4.0, args.cpu_seconds / 3), 1, seed=5)
        line["cpu_baseline"]["single_thread"] = {"value": v1_, "unit": UNIT, "sample": s1}
        line["parity"] = sampled_parity(FD, grid, model, out64, dm, dev, sel, port_rows)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_e2e(args, F, FD, w2, grid, model, dev, stream, flush, world, rank, v0, v1):
    """e2e through the public API: Field.build from PINNED host landmarks (H2D inside the timed
    region; with N ranks the process_group build broadcasts them from rank 0), the field stays
    on the device (what the GPU queries use), a D2H checksum of it ends the step.  e2e_export
    adds what the reference's Field.build hands back: the reference-layout factors (kinv @ S,
    36 per block, FP64) exported and copied to pinned host memory."""
    import torch
    import torch.distributed as dist

    pts_host = torch.tensor(w2.points).pin_memory()
    pg = dist.group.WORLD if world > 1 else None
    res = {}
    for export in (False, True):
        host_out = None
        if export:
            host_out = torch.empty(((v1 - v0), model.n_v * 36), dtype=torch.float64).pin_memory()
        times = []
        for i in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if export and world == 1:
                # the reference's build returns host factors: z-slab chunks, each chunk's export
                # and D2H overlapping the next chunk's build (Field.build(host_factors=True))
                fld = F.Field.build(pts_host, grid, model, "info", device=dev, host_factors=True, host_out=host_out)
                d2h = host_out.numel() * 8
            else:
                fld = F.Field.build(pts_host, grid, model, "info", device=dev, process_group=pg, replicate=False)
            if export and world > 1:
                fld.export_reference_to(host_out)
                d2h = host_out.numel() * 8
            elif not export:
                chk = fld.storage["f32"].sum(dtype=torch.float64).to("cpu", non_blocking=True)
                d2h = 8
            b.record(stream)
            b.synchronize()
            if i >= args.warmup:
                times.append(a.elapsed_time(b))
            del fld
        ms = float(np.mean(times))
        if world > 1:
            tt = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        tot_pairs = grid.voxel_count * w2.points.shape[0]
        res[export] = {"value": tot_pairs / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(pts_host.numel() * 8),
                       "d2h_bytes_per_step": int(d2h), "ms_per_step": ms,
                       "path": ("Field.build(pinned host landmarks, host_factors=True): z-slab chunks, each chunk's "
                                "export_reference (kinv @ S, reference layout FP64) and D2H into pinned host memory "
                                "overlapping the next chunk's build" if export else
                                "Field.build(pinned host landmarks) -> device-resident field (the GPU queries' "
                                "operand) -> D2H checksum")}
        del host_out
    return res[False], res[True]


def sampled_parity(FD, grid, model, out64, dm, dev, sel, port_rows):
    """The timed build's rows for the CPU-baseline sample voxels against the CPU port's rows
    for the same voxels (reference layout, max |delta| / voxel Frobenius norm; tolerance 1e-4)."""
    import torch

    from paper_2008_03324_b200 import _lib

    idx = torch.as_tensor(grid.internal_index(grid.index3_of(sel)), device=dev)
    src = out64[idx].contiguous()
    ref_dev = torch.empty((src.shape[0], model.n_v * 36), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().fif_export_reference(_lib.KIND_INFO, dm.c, src.data_ptr(), src.shape[0],
                                                ref_dev.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
               "fif_export_reference")
    mine = ref_dev.cpu().numpy()
    err = np.abs(mine - port_rows).max(axis=1) / np.maximum(np.linalg.norm(port_rows, axis=1), 1e-300)
    return {"voxels": int(len(sel)), "max_entry_over_voxel_frobenius": float(err.max()),
            "median": float(np.median(err)), "tol": 1e-4, "ok": bool(err.max() <= 1e-4),
            "against": "the CPU port's rows for the cpu_baseline sample (reference algorithm, FP64)"}


def _time(stream, fn, reps, flush=None):
    import torch

    times = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    return float(np.mean(times))


def secondary(args, F, FD, SC, w2, grid, model, pts, dev, stream, flush, world, rank, peaks, sms, max_mhz):
    import torch

    from paper_2008_03324_b200.parallel import slab_range

    res = {}
    hbm = float(peaks.get("hbm_gbs", 6550.4))
    fp32_peak = sms * 128 * 2 * max_mhz * 1e6 / 1e12
    reps = max(3, args.steps)
    # ── config-2 queries: replicated field, queries sharded ──
    fld = F.Field.build(pts, grid, model, "info", device=dev)
    q0, q1 = slab_range(w2.positions.shape[0], world, rank)
    pos = torch.tensor(w2.positions[q0:q1], device=dev)
    ax = torch.tensor(np.ascontiguousarray(w2.rotations[q0:q1, :, 2]), device=dev)
    out = {}
    run_q = lambda: fld.query_device(pos, ax, "trilinear", trace=True, full=True, grad=True, out=out)  # noqa: E731
    run_q()
    qms = _time(stream, run_q, reps, flush)
    q_traffic = None
    try:  # ncu dram bytes of the query kernels per query (profiles/ncu_summary.json)
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        q_traffic = prof["query_per_query"]["dram_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    nq = q1 - q0
    ns = model.n_v
    bytes_q = 8 * (QUERY_ROW_BYTES_GP_INFO(ns) + QUERY_TRACE_ROW_BYTES(ns)) + 48 + 8 * (1 + 6 + 36 + 216)
    res["query"] = {
        "workload": "config2: 100000 poses, trilinear, full 6x6 + trace + analytic d/d[t;theta], GP-70 info field",
        "value": nq * world / (qms / 1e3), "unit": "queries/s", "ms": qms,
        "roofline": {"bound": "hbm", "achieved": nq * bytes_q / (qms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": nq * bytes_q / (qms / 1e3) / 1e9 / hbm, "traffic": q_traffic,
                     "bytes_per_query": bytes_q,
                     "bytes_note": "8 corners x (FP32 S row 21 x N_s x 4 B + FP64 trace-table row N_s x 8 B) + "
                                   "pose + outputs (trace, 6x6, their gradients) in FP64"},
    }
    # ── config-3 point cloud + FIF on the same poses ──
    npose = 1000000
    w3 = SC.config3(npose)
    p0, p1 = slab_range(npose, world, rank)
    r = torch.tensor(w3.rotations[p0:p1].reshape(-1, 9), device=dev)
    t = torch.tensor(w3.positions[p0:p1], device=dev)
    cam = F.PinholeCamera.from_fov()
    outpc = torch.empty((p1 - p0, 36), dtype=torch.float64, device=dev)
    run_pc = lambda: F.exact_pose_fim_batch_device(r, t, pts, cam, out=outpc)  # noqa: E731
    run_pc()
    pms = _time(stream, run_pc, max(1, reps // 2))
    # visible fraction (needed for the roofline's per-pair count) from a 4 000-pose mask sample
    ns_vis = min(4000, p1 - p0)
    vmask = torch.zeros((ns_vis, pts.shape[0]), dtype=torch.uint8, device=dev)
    F.exact_pose_fim_batch_device(r[:ns_vis].contiguous(), t[:ns_vis].contiguous(), pts, cam, mask=vmask)
    vis = float(vmask.float().mean().item())
    del vmask
    pairs_pc = (p1 - p0) * pts.shape[0]
    flops_pair = PC_FLOPS_TEST + PC_FLOPS_VISIBLE * vis
    pc_ach = pairs_pc * flops_pair / (pms / 1e3) / 1e12
    res["pc"] = {"workload": "config3: 1e6 poses x 20000 landmarks, exact pinhole FIM (trace + 6x6)",
                 "value": pairs_pc * world / (pms / 1e3), "unit": "pose-landmark pairs/s", "ms": pms,
                 "visible_fraction": vis,
                 "roofline": {"bound": "fp32", "achieved": pc_ach, "peak": fp32_peak, "unit": "TFLOP/s",
                              "frac": pc_ach / fp32_peak, "kernel": "k_pc_fim",
                              "flops_per_pair": flops_pair,
                              "count": f"SURVEY 8(d): {PC_FLOPS_TEST} flop visibility test + {PC_FLOPS_VISIBLE} flop "
                                       f"6x6 accumulation x visible fraction {vis:.4f} (the reference's algorithm "
                                       "tests every pair; here groups of 32 Morton-ordered landmarks whose box is "
                                       "certainly outside / inside the view skip the per-landmark test, so the "
                                       "algorithmic rate can exceed what the test work alone would allow); the "
                                       "exact FP64 test inside the FP32 pre-test's margin is not counted"}}
    res["pc_vs_fif"] = pc_vs_fif(F, w3, p0, p1, fld, pts, outpc, dev, stream, reps, pms, model, grid)
    # ── masked build: range + occlusion gates fused into the build kernels ──
    if world == 1:
        res["masked_build"] = masked_build(F, FD, w2, grid, model, pts, dev, stream, reps)
    return res


def pc_vs_fif(F, w3, p0, p1, fld, pts, outpc, dev, stream, reps, pms, model, grid):
    """N1 / BASELINE configs[2]: FIF queries on the same config-3 poses as the point-cloud
    kernel (one device), and the FIF-vs-exact error in the style of the paper's Table II
    (relative Frobenius norm of the 6x6 and relative trace error, median and p90)."""
    import torch

    q = p1 - p0
    pos = torch.tensor(w3.positions[p0:p1], device=dev)
    ax = torch.tensor(np.ascontiguousarray(w3.rotations[p0:p1, :, 2]), device=dev)
    quad = F.build_quad_model()
    fq = F.Field.build(pts, grid, quad, "info", device=dev)
    out = {}
    for name, f in (("gp70", fld), ("quad", fq)):
        o = {}
        run = lambda: f.query_device(pos, ax, "trilinear", trace=True, full=True, out=o)  # noqa: E731
        run()
        ms = _time(stream, run, reps)
        fim = o["fim"]
        ok = o["status"] == 0
        d = (fim - outpc).reshape(q, 36)
        nf = torch.linalg.norm(outpc.reshape(q, 36), dim=1)
        rel = (torch.linalg.norm(d, dim=1) / torch.clamp(nf, min=1e-300))[ok & (nf > 0)]
        trp = outpc.reshape(q, 6, 6).diagonal(dim1=1, dim2=2).sum(-1)
        tre = (torch.abs(o["trace"] - trp) / torch.clamp(trp, min=1e-300))[ok & (trp > 0)]
        qs = torch.tensor([0.5, 0.9], dtype=torch.float64, device=dev)
        rq = torch.quantile(rel[:1_000_000].double(), qs).tolist() if rel.numel() else [None, None]
        tq = torch.quantile(tre[:1_000_000].double(), qs).tolist() if tre.numel() else [None, None]
        out[name] = {"ms": ms, "queries_per_s": q / (ms / 1e3), "speedup_vs_pc": pms / ms,
                     "in_field_fraction": float(ok.float().mean().item()),
                     "rel_fro_6x6": {"median": rq[0], "p90": rq[1]}, "rel_trace": {"median": tq[0], "p90": tq[1]}}
    return {"workload": f"{q} config-3 poses: exact point-cloud FIM (k_pc_fim, {pms:.2f} ms) vs FIF queries "
                        "(trilinear, full 6x6 + trace) on the config-2 fields; errors of FIF against the exact FIM",
            "pc_ms": pms, **out}


def masked_build(F, FD, w2, grid, model, pts, dev, stream, reps):
    """(f)3: config-2 GP-70 info build with range gates and an occluding pillar, the gates
    evaluated inside the build kernels (no (V, N) mask); occupancy pass + build timed."""
    import torch

    class _Box:
        def __init__(self, lo, hi):
            self.lo, self.hi = np.asarray(lo, float), np.asarray(hi, float)

    class _World:
        spheres = []
        boxes = [_Box([-1.0, -1.0, 0.0], [1.0, 1.0, 5.0])]

    mt = F.Matchability(d_near=0.25, d_far=8.0, occluders=_World())
    run = lambda: F.Field.build(pts, grid, model, "info", matchability=mt, device=dev)  # noqa: E731
    f = run()
    ms = _time(stream, run, max(2, reps // 3))
    cen = FD.device_centers(grid, dev)
    n_any = int(mt.device_any(cen, pts).sum().item())
    return {"workload": "config2 GP-70 info build, Matchability(d_near=0.25, d_far=8.0, occluders=2x2x5 m pillar) "
                        "fused into the build kernels",
            "ms": ms, "occupied_voxels": n_any, "rows": f.rows, "unit": "ms",
            "mask_bytes_avoided": int(grid.voxel_count * pts.shape[0])}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())

"""Side-by-side key metrics of ncu reports: python tools/ncu_cmp.py A.ncu-rep B.ncu-rep ..."""
import csv, io, subprocess, sys
keys = ["gpu__time_duration.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread"]
stall = "smsp__average_warps_issue_stalled_"
reps = sys.argv[1:]
vals = []
for r in reps:
    rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", r, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
    vals.append(dict(zip(rows[0], rows[2])))
names = keys + sorted(k for k in vals[0] if k.startswith(stall) and k.endswith("_per_issue_active.ratio"))
for k in names:
    xs = [v.get(k, "") for v in vals]
    if all(x in ("", "0", "0.000000") for x in xs):
        continue
    print(f"{k.replace(stall, 'stall_').replace('_per_issue_active.ratio', ''):70s} " + "  ".join(f"{x:>14s}" for x in xs))

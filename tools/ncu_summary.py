"""Summarise an ncu report: key SOL / occupancy / pipe metrics and top stall reasons."""
import csv, io, subprocess, sys

def run(rep, page, kernel=None, extra=()):
    cmd = ["ncu", "-i", rep, "--page", page, "--csv", *extra]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    return list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))

def main(rep, kernel=None):
    r = run(rep, "details", kernel)
    hdr = r[0]
    want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Theoretical Occupancy", "Achieved Active Warps Per SM",
            "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Executed Instructions", "Compute (SM) Throughput",
            "L1/TEX Cache Throughput", "DRAM Throughput", "Memory Throughput", "Block Limit Registers", "Block Limit Shared Mem",
            "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
    seen = {}
    for row in r[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in want and d["Metric Name"] not in seen:
            seen[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}"
    for k in want:
        if k in seen:
            print(f"  {k:38s} {seen[k]}")
    raw = run(rep, "raw", kernel)
    hdr, units, vals = raw[0], raw[1], raw[2]
    stalls = []
    keys = {}
    for h, v in zip(hdr, vals):
        if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        u = units[hdr.index(h)] if h in hdr else ""
        for k in ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                  "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                  "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"):
            if h.startswith(k) and h not in keys:
                keys[h] = f"{v} {u}"
    for h, v in keys.items():
        print(f"  {h:60s} {v}")
    tot = sum(v for v, _ in stalls) or 1
    print("  stalls: " + ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(stalls, reverse=True)[:8]))

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)

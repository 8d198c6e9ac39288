"""Per-instruction hot spots of an ncu report (source page, SASS): top instructions by
executed count and by stall samples, plus totals by opcode.  Usage: ncu_hot.py REP [N]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def f(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0
tot_ex = sum(f(d["Instructions Executed"]) for d in data)
tot_st = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
print(f"total warp instructions {tot_ex:.4g}, stall samples {tot_st:.4g}")
by_op = defaultdict(lambda: [0.0, 0.0])
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    op = op.split(".")[0]
    by_op[op][0] += f(d["Instructions Executed"])
    by_op[op][1] += f(d["Warp Stall Sampling (All Samples)"])
print("by opcode (executed %, stall %):")
for op, (e, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"  {op:12s} {100*e/tot_ex:6.2f}%  {100*s/tot_st:6.2f}%")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("top stall instructions:")
for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:n]:
    st = sorted(((f(d[c]), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"  {d['Address']:>6s} {d['Source'][:60]:60s} {100*f(d['Warp Stall Sampling (All Samples)'])/tot_st:5.2f}%  "
          + " ".join(f"{c}={v:.0f}" for v, c in st if v))

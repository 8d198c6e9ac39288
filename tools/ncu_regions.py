"""Stall samples of an ncu report (source page, SASS) grouped into the regions between
synchronisation instructions, plus the hottest instructions.  Usage: ncu_regions.py REP [MINPCT]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
minpct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
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


tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
KEYS = ("BAR.", "LDTM", "UTCBAR", "SYNCS.PHASECHK", "UTCHMMA")
acc, acc_i, start = 0.0, 0.0, 0
for i, d in enumerate(data):
    s = f(d["Warp Stall Sampling (All Samples)"])
    src = d["Source"]
    key = any(k in src for k in KEYS)
    if key and acc > 0:
        print(f"  [{start:5d}-{i:5d}) region stall {100 * acc / tot:5.2f}%  instr {acc_i:.3g}")
        acc, acc_i, start = 0.0, 0.0, i
    acc += s
    acc_i += f(d["Instructions Executed"])
    if 100 * s / tot >= minpct or (key and "UTCHMMA" not in src):
        st = sorted(((f(d[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(i, f"{100 * s / tot:5.2f}%", f"{f(d['Instructions Executed']):.3g}", src[:70],
              " ".join(f"{c}={v:.0f}" for v, c in st if v))
print(f"  [{start:5d}-{len(data):5d}) region stall {100 * acc / tot:5.2f}%")

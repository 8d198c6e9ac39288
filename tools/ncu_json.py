"""Write profiles/ncu_summary.json (the `traffic` figures bench.py reports) from the
--set full captures tools/round_measure.sh leaves in gpurun_out/."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")


def raw(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kernel}"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = r[0], r[1], r[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1,
             "usecond": 1e-3, "msecond": 1, "nsecond": 1e-6}
    def get(name):
        i = hdr.index(name)
        return float(vals[i].replace(",", "")) * scale.get(units[i], 1)
    return {"dram_read": get("dram__bytes_read.sum"), "dram_write": get("dram__bytes_write.sum"),
            "duration_ms_under_ncu": get("gpu__time_duration.sum")}


res = {}
gi = raw(os.path.join(O, "full_k_gp_info_h16.ncu-rep"), "k_gp_info_h16")
gi["dram_bytes_per_launch"] = gi["dram_read"] + gi["dram_write"]
gi["source"] = "ncu --set full capture of bench.py, one k_gp_info_h16 launch (config-2 GP-70 info build)"
res["k_gp_info_h16"] = gi
q = raw(os.path.join(O, "full_k_query_info.ncu-rep"), "k_query_info")
p = raw(os.path.join(O, "full_k_query_prep_gp.ncu-rep"), "k_query_prep_gp")
res["k_query_info"], res["k_query_prep_gp"] = q, p
nq = 100000
res["query_per_query"] = {"dram_bytes": (q["dram_read"] + q["dram_write"] + p["dram_read"] + p["dram_write"]) / nq,
                          "source": "k_query_prep_gp + k_query_info dram bytes / 1e5 queries (bench.py config-2)"}
path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "ncu_summary.json")
json.dump(res, open(path, "w"), indent=1)
print(json.dumps(res, indent=1))

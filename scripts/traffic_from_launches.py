"""profiles/roofline_traffic.json from an ncu launch list (dram__bytes_read/write.sum per
launch): DRAM bytes per point-stage and per point-step of the fused stage kernels, the
`traffic` field of bench.py's roofline (per launch = per point-stage x local points).
  python scripts/traffic_from_launches.py LAUNCHES.csv NPOINTS WORKLOAD [out.json]"""
import csv
import json
import sys

path, npts, wl = sys.argv[1], float(sys.argv[2]), sys.argv[3]
out = sys.argv[4] if len(sys.argv) > 4 else "profiles/roofline_traffic.json"
S = 16 if wl.endswith("c128") else 8  # bytes per complex (C4 and *_c64: complex64)
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi or not r[ki].startswith(("void stage_stream_kernel", "void line_stream_kernel")):
        continue
    per.setdefault(r[idi], {})[r[mi]] = float(r[vi].replace(",", ""))
launches = [v for v in per.values() if "dram__bytes_read.sum" in v]
tot = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in launches)
bps = tot / len(launches) / npts
res = {"workload": wl, "source": f"{path} (ncu dram__bytes_read/write.sum, {len(launches)} stage launches)",
       "dram_bytes_per_point_stage": round(bps, 4), "dram_bytes_per_point_step": round(4 * bps, 2),
       "algorithmic_bytes_per_point_step_16S": 16 * S, "moved_by_design_12S": 12 * S}
# the file keeps the bench workload (C4) at top level and every other measured workload under
# "workloads" (key = WORKLOAD or WORKLOAD_dtype, as bench.py looks them up)
import os

cur = json.load(open(out)) if os.path.exists(out) else {}
if wl == "C4" or not cur:
    keep = cur.get("workloads", {})
    cur = dict(res)
    cur["workloads"] = keep
else:
    cur.setdefault("workloads", {})[wl] = res
json.dump(cur, open(out, "w"), indent=1)
print(json.dumps(res))

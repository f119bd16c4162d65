"""profiles/roofline_traffic.json from an ncu launch list (dram__bytes_read/write.sum per
launch): DRAM bytes per point-stage and per point-step of the fused stage kernels, the
`traffic` field of bench.py's roofline (per launch = per point-stage x local points).
  python scripts/traffic_from_launches.py LAUNCHES.csv NPOINTS WORKLOAD [out.json]"""
import csv
import json
import sys

path, npts, wl = sys.argv[1], float(sys.argv[2]), sys.argv[3]
out = sys.argv[4] if len(sys.argv) > 4 else "profiles/roofline_traffic.json"
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi or not r[ki].startswith("void stage_stream_kernel"):
        continue
    per.setdefault(r[idi], {})[r[mi]] = float(r[vi].replace(",", ""))
launches = [v for v in per.values() if "dram__bytes_read.sum" in v]
tot = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in launches)
bps = tot / len(launches) / npts
res = {"workload": wl, "source": f"{path} (ncu dram__bytes_read/write.sum, {len(launches)} stage launches)",
       "dram_bytes_per_point_stage": round(bps, 4), "dram_bytes_per_point_step": round(4 * bps, 2),
       "algorithmic_bytes_per_point_step_16S": 128, "moved_by_design_12S": 96}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))

"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel
and by z-line op: launches, total time and share.  Usage:
python tools/launch_summary.py gpurun_out/launches.csv "<command>" > profiles/<name>.json"""
import collections
import csv
import json
import re
import sys

OPS = ["realize", "map", "map_tc", "map_tf", "inv_vol", "bwd_vol", "outer", "outer_pair", "contract"]
rows = list(csv.reader(open(sys.argv[1])))
agg = collections.defaultdict(lambda: [0, 0.0])
ki = vi = ui = None
scale = 1.0
for r in rows:
    if "Kernel Name" in r:
        ki, vi, ui = r.index("Kernel Name"), r.index("Metric Value"), r.index("Metric Unit")
        continue
    if ki is None or len(r) <= vi or not r[vi]:
        continue
    name = r[ki]
    unit = r[ui]
    t = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    m = re.search(r"k_zlines<(\w+), (?:blr::)?WShape<[^>]*>, (?:\(int\))?(\d)>", name)
    if m:
        key = f"k_zlines[{OPS[int(m.group(2))]}]"
    else:
        key = re.sub(r"^void ", "", name).split("<")[0].split("(")[0].replace("blr::", "")
    agg[key][0] += 1
    agg[key][1] += t
tot = sum(v[1] for v in agg.values())
out = {"command": sys.argv[2] if len(sys.argv) > 2 else "",
       "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache serialized per-launch times; compare shares, not absolutes",
       "total_us": round(tot, 1),
       "kernels": {k: {"launches": v[0], "total_us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2),
                       "share": round(v[1] / tot, 4)}
                   for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
print(json.dumps(out, indent=1))

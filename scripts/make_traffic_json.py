"""Collect per-launch DRAM traffic of the stage kernels from ncu CSVs
(gpurun_out/traffic_<kind>_n<N>.csv, made by scripts/gpu_final_sweep.sh) into
profiles/ncu_traffic.json, which bench.py reports as roofline.traffic."""
import csv
import glob
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "traffic_*_n*.csv"))):
    kind, n = re.match(r"traffic_(\w+)_n(\d+)\.csv", os.path.basename(path)).groups()
    rows = [r for r in csv.reader(open(path)) if r and (r[0] == "ID" or r[0].isdigit())]
    if len(rows) < 2:
        continue
    h = rows[0]
    vals = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d.get("Metric Name")
        unit = d.get("Metric Unit", "")
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3}.get(unit, 1)
        vals[name] = v * scale
        vals["kernel"] = d.get("Kernel Name", "")
    if "dram__bytes_read.sum" not in vals:
        continue
    out.setdefault(kind, {})[n] = {
        "bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
        "read": vals["dram__bytes_read.sum"], "write": vals["dram__bytes_write.sum"],
        "duration_s_ncu": vals.get("gpu__time_duration.sum"), "kernel": vals["kernel"][:80],
        "capture": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                   "-s 16 -c 1 (stage 2 of step 4; serialised, cold clocks)",
    }
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1, sort_keys=True)
print(json.dumps({k: {n: round(v["bytes_per_launch"] / 1e9, 3) for n, v in d.items()} for k, d in out.items()}))

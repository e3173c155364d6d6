"""Update profiles/ncu_traffic.json (bench.py's roofline.traffic) from ncu --set full captures of a
measurement run: gpurun_out/<tag>_full_n<N>.ncu-rep (exact wedge kernel), <tag>_tet4.ncu-rep (tet
kernel, N = 4), <tag>_wadg5.ncu-rep (WADG wedge kernel, N = 5).  Entries not captured are kept.
usage: traffic_from_reps.py TAG"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
out = json.load(open(path))


def metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, r = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}

    def get(name):
        i = h.index(name)
        return float(r[i].replace(",", "")) * scale.get(units[i], 1)
    return {"read": get("dram__bytes_read.sum"), "write": get("dram__bytes_write.sum"),
            "duration_s_ncu": get("gpu__time_duration.sum"), "kernel": r[h.index("Kernel Name")][:80]}


caps = [("exact", str(n), f"{tag}_full_n{n}") for n in range(1, 8)] + [("tet", "4", f"{tag}_tet4"),
                                                                      ("wadg", "5", f"{tag}_wadg5")]
for kind, n, name in caps:
    rep = os.path.join(ROOT, "gpurun_out", name + ".ncu-rep")
    if not os.path.exists(rep):
        continue
    m = metrics(rep)
    out.setdefault(kind, {})[n] = {
        "bytes_per_launch": m["read"] + m["write"], "read": m["read"], "write": m["write"],
        "duration_s_ncu": m["duration_s_ncu"], "kernel": m["kernel"],
        "capture": f"ncu --set full --clock-control none -s 16 -c 1 ({name}.ncu-rep; serialised, cold clocks)"}
json.dump(out, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps({k: {n: round(v["bytes_per_launch"] / 1e9, 3) for n, v in d.items()} for k, d in out.items()}))

"""Per-source-line instruction counts and stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname = None
agg = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] in ("", "Function Name"):
        continue
    if r[0] == "" or not r[0].isdigit():
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")])
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    agg.append((fname, int(r[0]), r[1][:90], inst, samp))
ti = sum(a[3] for a in agg) or 1
ts = sum(a[4] for a in agg) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = 4 if len(sys.argv) > 3 and sys.argv[3] == "samples" else 3
for f, ln, src, inst, samp in sorted(agg, key=lambda a: -a[key])[:top]:
    print(f"{f[:14]:14s}:{ln:4d} inst {100*inst/ti:5.1f}% stall {100*samp/ts:5.1f}%  {src}")

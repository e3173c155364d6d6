#!/usr/bin/env python3
"""SASS instruction histogram per kernel of the built library (cuobjdump -sass):
evidence of the FP64 tensor-core (DMMA), bulk-TMA (UBLKCP) and mbarrier (SYNCS)
paths, and that no tcgen05 (UTC*MMA / LDTM / STTM) or 2D TMA (UTMALDG) is used."""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1607_03399_b200/_lib/libprismdg_b200.so"
WATCH = ["DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "LDG", "STG", "SHFL",
         "BAR", "UTCHMMA", "UTCMMA", "UTMALDG", "LDTM", "STTM"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for ln in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", ln)
    if m and kern:
        counts[kern][m.group(2)] += 1
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print(f"# SASS histogram of {LIB} ({len(counts)} kernels), static instruction counts")
print("total: " + ", ".join(f"{w} {tot.get(w, 0)}" for w in WATCH))
demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
for (k, c), name in zip(counts.items(), demangle):
    short = re.sub(r"pdg::\(anonymous namespace\)::", "", name)
    short = re.sub(r"\(pdg::\w+\)", "", short)
    if any(s in short for s in ("wedge_", "tet_")):
        print(f"{short[:70]:70s} " + " ".join(f"{w}:{c[w]}" for w in WATCH if c.get(w)))

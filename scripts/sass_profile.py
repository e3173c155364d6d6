#!/usr/bin/env python3
"""Summarise an ncu --page source --print-source sass CSV export: stall samples
and L1 shared wavefronts by opcode, the hottest instructions, and the SASS
instruction mix (DMMA / LDS / STS / LDG / STG / UBLKCP ...)."""
import csv
import re
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]

    def num(r, k):
        try:
            return float(r[idx[k]])
        except (ValueError, KeyError):
            return 0.0

    by_op = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    stalls = defaultdict(float)
    tot_samples = 0.0
    for r in data:
        src = r[idx["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
        base = op.split(".")[0]
        e = by_op[base]
        e[0] += 1
        e[1] += num(r, "Warp Stall Sampling (All Samples)")
        e[2] += num(r, "L1 Wavefronts Shared")
        e[3] += num(r, "L1 Wavefronts Shared Excessive")
        e[4] += num(r, "Instructions Executed")
        tot_samples += num(r, "Warp Stall Sampling (All Samples)")
        for c in stall_cols:
            stalls[c] += num(r, c)
    print(f"{'opcode':10s} {'count':>6s} {'samples%':>9s} {'wf_shared':>12s} {'excess':>11s} {'executed':>12s}")
    for op, e in sorted(by_op.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{op:10s} {e[0]:6d} {100 * e[1] / max(tot_samples, 1):8.1f}% {e[2]:12.0f} {e[3]:11.0f} {e[4]:12.0f}")
    print("\nstall reasons (all samples):")
    for c, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {c:24s} {100 * v / max(tot_samples, 1):5.1f}%")
    print(f"\nhottest {top} instructions:")
    hot = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]
    for r in hot:
        s = num(r, "Warp Stall Sampling (All Samples)")
        top3 = sorted(((num(r, c), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"  {100 * s / tot_samples:5.2f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} "
              f"wf={num(r, 'L1 Wavefronts Shared'):.0f} " + " ".join(f"{c}:{100 * v / max(s, 1):.0f}%" for v, c in top3))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

#!/usr/bin/env python3
"""One row per .ncu-rep (one stage-kernel launch each): time, DRAM bytes vs the
algorithmic bytes, occupancy, issue, L1 / DMMA / FP64 pipe use, top stalls."""
import csv
import re
import subprocess
import sys


def alg_bytes(N, wedges=1_000_000, later=True):
    nq, nt = N + 1, (N + 1) * (N + 2) // 2
    np_ = nq * nt
    return wedges * (8 * ((16 if later else 12) * np_ + nt * nt + 3 * nt * nq + 34 + 2 * nq) + 48)


def row(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    d = dict(zip(h, v))
    f = lambda k: float(d.get(k) or "nan")
    pre = "smsp__average_warps_issue_stalled_"
    st = {k[len(pre):].replace("_per_issue_active.ratio", ""): float(d[k]) for k in d
          if k.startswith(pre) and d[k] not in ("", "n/a")}
    tot = sum(st.values())
    top = ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])[:4])
    name = d.get("Kernel Name", "?")
    m = re.search(r"<(\d+)", name)
    N = int(m.group(1)) if m else 0
    dram = (f("dram__bytes_read.sum") + f("dram__bytes_write.sum"))
    unit = d.get("dram__bytes_read.sum", "")
    t_ms = f("gpu__time_duration.sum")
    return (f"| {N} | `{name.split('(')[0].replace('void ', '')[:34]}` | {t_ms:.3f} | {f('launch__registers_per_thread'):.0f} | "
            f"{f('sm__warps_active.avg.pct_of_peak_sustained_active') * 0.64:.1f} | "
            f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f}% | "
            f"{f('l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f}% | "
            f"{f('sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active'):.0f}% | "
            f"{f('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f}% | {top} |")


if __name__ == "__main__":
    print("| N | kernel | ncu ms | regs | warps/SM | issue | L1 | DMMA pipe | FP64 pipe | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for rep in sys.argv[1:]:
        print(row(rep))

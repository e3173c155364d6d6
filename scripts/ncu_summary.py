"""Print stall breakdown and key counters of an .ncu-rep (single kernel)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(h, v))
pre = "smsp__average_warps_issue_stalled_"
st = {k[len(pre):].replace("_per_issue_active.ratio", ""): float(d[k]) for k in d
      if k.startswith(pre) and d[k] not in ("", "n/a")}
tot = sum(st.values())
print("stalls (warps per issue):", f"total {tot:.2f}")
for k, x in sorted(st.items(), key=lambda t: -t[1])[:9]:
    print(f"  {k:24s} {x:6.2f} {100 * x / tot:5.1f}%")
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    print(f"  {k:78s} {d.get(k)}")

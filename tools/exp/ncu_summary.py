"""Key metrics + stall breakdown per kernel launch of an ncu report.
  python tools/exp/ncu_summary.py <rep>"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[0], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__warps_active.avg.per_cycle_active"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w[:60]:60s}", [r[i][:40] for r in data])
st = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued")]
for r in data:
    tot = sum(float(r[h.index(c)] or 0) for c in st)
    top = sorted(((c.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[h.index(c)] or 0) / tot)
                  for c in st), key=lambda x: -x[1])[:8]
    print("  stalls:", " ".join(f"{k}={v * 100:.0f}%" for k, v in top))

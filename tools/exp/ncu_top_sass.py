"""Top SASS instructions by warp-stall samples in one kernel of an ncu report.
  python tools/exp/ncu_top_sass.py <rep> <launch-skip> [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, skip = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][1][:120])
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = []
for r in rows[2:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break
    data.append(r)
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
by_op = defaultdict(lambda: [0, 0])
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    by_op[op.split(".")[0]][0] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    by_op[op.split(".")[0]][1] += int(r[ix["Instructions Executed"]] or 0)
print("samples", tot)
for op, (s, n) in sorted(by_op.items(), key=lambda x: -x[1][0])[:20]:
    print(f"  {op:10s} samples {s / tot * 100:5.1f}%  inst {n}")
order = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
for i in order[:top]:
    r = data[i]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((k, int(r[ix[k]] or 0)) for k in stalls), key=lambda x: -x[1])[:2]
    print(f"{i:5d} {s / tot * 100:5.2f}% {r[ix['Source']].strip()[:60]:60s} " +
          " ".join(f"{k[6:]}={v}" for k, v in st))

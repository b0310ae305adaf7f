"""Summarise an ncu source page: stall totals, per-opcode counts per warp-tile."""
import csv
import subprocess
import sys

rep, warp_tiles = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: 0 for k in stalls}
allsamp = 0
ops = {}


def op(r):
    t = r[1].split()
    o = t[1] if t[0].startswith("@") else t[0]
    return o.split(".")[0]


for r in data:
    for k in stalls:
        try:
            tot[k] += int(r[ix[k]])
        except ValueError:
            pass
    allsamp += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    ops[op(r)] = ops.get(op(r), 0) + n
print("samples", allsamp, "inst/warp-tile", round(sum(ops.values()) / warp_tiles, 1))
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:25s} {v / allsamp * 100:5.1f}%")
print([(k, round(v / warp_tiles, 1)) for k, v in sorted(ops.items(), key=lambda x: -x[1])[:26]])

"""Join an ncu SASS source page with nvdisasm line info: per source line,
dynamic instructions per warp-tile and stall samples.

  python tools/exp/ncu_lines.py <rep> <cubin> <kernel-substring> <warp_tiles>
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, kname, wt = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(sass) if l.startswith(".text.") and kname in l)
loc = None
seq = []
for l in sass[start + 1:]:
    if l.startswith("//---") and ".text." in l:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        loc = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        seq.append((loc, l.strip()))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = rows[2:]
print("sass lines", len(seq), "ncu rows", len(data))
agg = defaultdict(lambda: [0, 0, defaultdict(int)])
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for (loc, _), r in zip(seq, data):
    a = agg[loc]
    a[0] += int(r[ix["Instructions Executed"]] or 0)
    a[1] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for k in stalls:
        try:
            a[2][k] += int(r[ix[k]])
        except ValueError:
            pass
tot = sum(a[1] for a in agg.values())
for loc, (n, smp, st) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    top = sorted(st.items(), key=lambda x: -x[1])[:2]
    print(f"{str(loc):34s} inst/wt {n / wt:7.1f}  samples {smp / tot * 100:5.1f}%  "
          + " ".join(f"{k[6:]}={v / tot * 100:.1f}" for k, v in top))

"""SASS instruction census of the library's kernels (cuobjdump -sass), for
profiles/: proves the tile movement (UTMALDG/UTMAPF/SYNCS = TMA + mbarrier,
LDGSTS = sm_80 cp.async) and the FP64 instruction mix per kernel.
   python tools/sass_summary.py [substring...] > profiles/sass_<round>.txt"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2001_10554_b200", "lib", "libqsb200.so")
OPS = ["UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDGSTS", "SYNCS", "LDS", "STS", "LDG", "STG",
       "DFMA", "DMUL", "DADD", "BAR", "SHFL"]


def main():
    want = sys.argv[1:] or ["k_"]
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*Function : ", txt)
    print(f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)}: opcode counts per kernel")
    print("kernel".ljust(40) + "".join(o.rjust(8) for o in OPS))
    for f in parts[1:]:
        name = f.split("\n", 1)[0].strip()
        m = re.search(r"(k_\w+?)I|(k_\w+?)E", name)
        short = (m.group(1) or m.group(2)) if m else name
        tmpl = re.search(r"ILb(\d)ELb(\d)", name)
        if tmpl:
            short += f"<{tmpl.group(1)},{tmpl.group(2)}>"
        if not any(w in name for w in want):
            continue
        body = [ln for ln in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln)]
        cnt = {o: sum(1 for ln in body if re.search(r"\b" + o + r"(\.|\s|$)", ln)) for o in OPS}
        print(short[:40].ljust(40) + "".join(str(cnt[o]).rjust(8) for o in OPS))


if __name__ == "__main__":
    main()

"""Build experimental variants of libqsb200.so (tile-shape macros) into
tools/exp/variants/<name>/ so one gpurun call can time them all
(QSB_LIB=<path> selects a variant at load time)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import build as B  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
VARIANTS = {
    # default build: one 256-thread group per CTA, two CTAs per SM, 2^12 tiles
    "base": [],
    # the round-1 variants (results in profiles/r01_notes.md); GROUPS=2 means the
    # ping-pong pair of groups in one CTA
    "t11g2": ["-DQSB_TILE_LOG2=11", "-DQSB_TILE_GROUPS=2", "-DQSB_TILE_MINB=1"],
    "r3t11": ["-DQSB_REG_LOG2=3", "-DQSB_TILE_LOG2=11", "-DQSB_TILE_GROUPS=2",
              "-DQSB_TILE_MINB=1"],
    "t11g1m2": ["-DQSB_TILE_LOG2=11", "-DQSB_TILE_GROUPS=1", "-DQSB_TILE_MINB=2"],
    "t11np": ["-DQSB_TILE_LOG2=11", "-DQSB_TILE_GROUPS=2", "-DQSB_TILE_MINB=1",
              "-DQSB_NO_PINGPONG"],
    "t10g2": ["-DQSB_TILE_LOG2=10", "-DQSB_TILE_GROUPS=2", "-DQSB_TILE_MINB=1"],
    "g1": ["-DQSB_TILE_GROUPS=1", "-DQSB_TILE_MINB=1"],
    "g1m2": ["-DQSB_TILE_GROUPS=1", "-DQSB_TILE_MINB=2"],
    "t11g1m4": ["-DQSB_TILE_LOG2=11", "-DQSB_TILE_GROUPS=1", "-DQSB_TILE_MINB=4"],
    "t11g1m3": ["-DQSB_TILE_LOG2=11", "-DQSB_TILE_GROUPS=1", "-DQSB_TILE_MINB=3"],
    "pp": ["-DQSB_TILE_GROUPS=2", "-DQSB_TILE_MINB=1"],
    "low2": ["-DQSB_LOW_BITS=2"],
    "prof": ["-DQSB_PROF"],
    "t11dbuf2": ["-DQSB_DBUF", "-DQSB_TILE_LOG2=11", "-DQSB_TILE_MINB=2"],
    "t11dbuf3": ["-DQSB_DBUF", "-DQSB_TILE_LOG2=11", "-DQSB_TILE_MINB=3"],
    "t11m3": ["-DQSB_TILE_LOG2=11", "-DQSB_TILE_MINB=3"],
    "nogmem": ["-DQSB_NO_GMEM"],
    "noloads": ["-DQSB_NO_LOADS"],
    "nostores": ["-DQSB_NO_STORES"],
    "nogmem_nosmem": ["-DQSB_NO_GMEM", "-DQSB_NO_SMEM_ROUND"],
    "r5": ["-DQSB_REG_LOG2=5"],
    "r5nogmem": ["-DQSB_REG_LOG2=5", "-DQSB_NO_GMEM"],
}


def main(names):
    def one(name):
        out = os.path.join(HERE, "variants", name, "libqsb200.so")
        B.build(out=out, extra_flags=VARIANTS[name])
        return name, out

    with ThreadPoolExecutor(len(names)) as ex:
        for name, out in ex.map(one, names):
            print(name, out)


if __name__ == "__main__":
    main(sys.argv[1:] or list(VARIANTS))

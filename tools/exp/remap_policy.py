"""Count swaps and passes per sweep step under qubit remapping (emulated ranks)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.circuit import GateSpec
from paper_2001_10554_b200.workloads import haar_2x2

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
m = 16
n = m + P.bit_length() - 1
rng = np.random.default_rng(0)
us = [[haar_2x2(rng) for _ in range(n)] for _ in range(6)]


def rank_fn(comm):
    ctx = runtime.make_context(comm, n, 1, 0, remap=True)
    ctx.norm_check_interval = 0
    out = []
    for stp in range(6):
        m0 = ctx.state.counters()[0]
        p0 = ctx.queue.passes_total
        for k in range(n):
            runtime.apply_gate(ctx, GateSpec("custom", (k,), matrix=us[stp][k]))
        ctx.flush()
        out.append(((ctx.state.counters()[0] - m0) // 2, ctx.queue.passes_total - p0))
    return out


res = runtime.run_spmd(P, rank_fn, timeout=120)
print(f"P={P} n={n}: (swaps, passes) per step:", res[0])

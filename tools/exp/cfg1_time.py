"""Config 1 (n=20 random circuit, 295 gates) end to end through the public API."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.circuit import Circuit
from paper_2001_10554_b200.workloads import config1_gates

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
circ = Circuit(n, tuple(config1_gates(n, 10, 20260809)))
for fuse in (True, False):
    ctx = runtime.make_context(None, n, fuse=fuse)
    runtime.run_circuit(ctx, circ)
    ctx.state.synchronize()
    times = []
    for _ in range(5):
        runtime.reset_state(ctx)
        t0 = time.perf_counter()
        runtime.run_circuit(ctx, circ)
        probs = [runtime.measure_probability(ctx, q) for q in range(n)]
        psi = ctx.state.download()
        times.append(time.perf_counter() - t0)
    print(f"n={n} fuse={fuse}: {np.median(times)*1e3:.2f} ms per circuit (+{n} probabilities + "
          f"state download), passes {ctx.queue.passes_total // 6}")

import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.circuit import Circuit
from paper_2001_10554_b200.workloads import config1_gates
n = 20
circ = Circuit(n, tuple(config1_gates(n, 10, 20260809)))
for fuse in (True, False):
    ctx = runtime.make_context(None, n, fuse=fuse)
    runtime.run_circuit(ctx, circ); ctx.state.synchronize()
    st = ctx.state
    st.launch_log(True)
    runtime.reset_state(ctx)
    t0 = time.perf_counter()
    runtime.run_circuit(ctx, circ)
    t1 = time.perf_counter()
    st.synchronize()
    t2 = time.perf_counter()
    ms, kinds = st.read_launch_log()
    st.launch_log(False)
    print(f"fuse={fuse}: host {1e3*(t1-t0):.2f} ms, until sync {1e3*(t2-t0):.2f} ms, device sum {ms.sum():.3f} ms over {len(ms)} launches")
ctx = runtime.make_context(None, n, fuse=True)
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    runtime.reset_state(ctx); runtime.run_circuit(ctx, circ)
ctx.state.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)

"""Host vs device time of one config-5 pool circuit (512 x n=20, p=4):
wall clock around runtime.run_circuit_pool (+ sync) vs the launch log.
  python tools/exp/qaoa_host.py [exact|factored]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import runtime  # noqa: E402
from paper_2001_10554_b200.circuit import build_qaoa_circuit, qaoa_bindings  # noqa: E402
from paper_2001_10554_b200.workloads import random_3regular_graph  # noqa: E402

S, n, p = 512, 20, 4
rng = np.random.default_rng(0)
g = random_3regular_graph(n, rng)
circ = build_qaoa_circuit(g, p)
fuse = "factored" if (sys.argv[1] if len(sys.argv) > 1 else "factored") == "factored" else True
ctx = runtime.make_context(None, n, num_states=S, fuse=fuse)
ctx.norm_check_interval = 0
for rep in range(4):
    pos = rng.uniform(0, np.pi, size=(S, 2 * p))
    t0 = time.perf_counter()
    tables = {}
    for s in range(S):
        for k, v in qaoa_bindings(p, pos[s]).items():
            tables.setdefault(k, np.empty(S))[s] = v
    t1 = time.perf_counter()
    ctx.state.launch_log(True)
    runtime.reset_state(ctx)
    runtime.run_circuit_pool(ctx, circ, tables)
    t2 = time.perf_counter()
    ctx.state.synchronize()
    t3 = time.perf_counter()
    ms, kinds = ctx.state.read_launch_log()
    ctx.state.launch_log(False)
    print(f"{sys.argv[1:]} tables {1e3 * (t1 - t0):.2f} ms, enqueue {1e3 * (t2 - t1):.2f} ms, "
          f"sync {1e3 * (t3 - t2):.2f} ms, device {float(ms.sum()):.2f} ms")

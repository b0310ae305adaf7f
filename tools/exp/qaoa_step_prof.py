"""Where a config-5 swarm step's wall time goes (GPU box): reset, host-side
program build + enqueue, device passes, <C>, PSO move; plus a cProfile of the
host side of run_circuit_pool."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import optimize as qopt, runtime  # noqa: E402
from paper_2001_10554_b200.circuit import build_qaoa_circuit  # noqa: E402
from paper_2001_10554_b200.noise import SCOPE_POOL, RandomStream  # noqa: E402

n, depth, S = 20, 4, 512
ps = RandomStream(20260809, SCOPE_POOL, 0)
graph = qopt.random_3regular_graph(n, ps.split(0))
circ = build_qaoa_circuit(graph, depth)
exact = qopt.exact_maxcut(graph)
swarm = qopt.init_swarm(S, 2 * depth, stream=ps.split(1))
ctx = runtime.make_context(None, n, S, 1, fuse="factored")
ctx.norm_check_interval = 0
st = ctx.state
edges = np.asarray(graph.edges, dtype=np.int32)
T = {}


def tick(name, t0):
    T.setdefault(name, []).append(1e3 * (time.perf_counter() - t0))
    return time.perf_counter()


def step(prof=None):
    t = time.perf_counter()
    pos = np.stack([p.position for p in swarm.particles])
    tabs = qopt.qaoa_slot_tables(pos, depth)
    t = tick("tables", t)
    runtime.reset_state(ctx)
    t = tick("reset_enqueue", t)
    if prof:
        prof.enable()
    runtime.run_circuit_pool(ctx, circ, tabs)
    if prof:
        prof.disable()
    t = tick("circuit_enqueue", t)
    st.synchronize()
    t = tick("device_wait", t)
    vals = ctx.pool.observable(3, 0, edges) / exact
    t = tick("observable", t)
    qopt.step_swarm(swarm, vals)
    tick("pso", t)


for _ in range(3):
    step()
T.clear()
prof = cProfile.Profile()
t0 = time.perf_counter()
for k in range(10):
    step(prof)
wall = 1e3 * (time.perf_counter() - t0) / 10
print({k: round(float(np.mean(v)), 3) for k, v in T.items()}, "wall/step", round(wall, 3))
pstats.Stats(prof).sort_stats("cumulative").print_stats(25)
pstats.Stats(prof).sort_stats("tottime").print_stats(15)

"""Per-pass timing of the config-5 pool circuit (512 x n=20, p=4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import runtime, _native as N
from paper_2001_10554_b200.circuit import build_qaoa_circuit, qaoa_bindings
from paper_2001_10554_b200.workloads import random_3regular_graph

S, n, p = 512, 20, 4
rng = np.random.default_rng(0)
g = random_3regular_graph(n, rng)
circ = build_qaoa_circuit(g, p)
pos = rng.uniform(0, np.pi, size=(S, 2 * p))
tables = {}
for s in range(S):
    for k, v in qaoa_bindings(p, pos[s]).items():
        tables.setdefault(k, np.empty(S))[s] = v
fuse = "factored" if (sys.argv[1] if len(sys.argv) > 1 else "exact") == "factored" else True
ctx = runtime.make_context(None, n, num_states=S, fuse=fuse)
ctx.norm_check_interval = 0  # diagnostics builds (QSB_EXP_*) break the norm on purpose
runtime.run_circuit_pool(ctx, circ, tables)
ctx.state.synchronize()
ctx.state.launch_log(True)
runtime.reset_state(ctx)
runtime.run_circuit_pool(ctx, circ, tables)
ms, kinds = ctx.state.read_launch_log()
print(sys.argv[1:], "total", round(float(ms.sum()), 2), "launches",
      list(zip(kinds.tolist(), np.round(ms, 3).tolist())))
q = runtime.GateQueue(ctx.state)
# plan of the same program
gates = []
for gs in circ.gates:
    if gs.kind == "diagcost":
        gates.append(N.QsGate(2, 0, -1, 0, 0, 0))
    else:
        gates.append(N.QsGate(0, gs.qubits[0], -1, 0, 0, 0))
print("plan starts", N.plan_program(n, gates))

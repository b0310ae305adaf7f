"""Randomised parity campaign: fused pool programs (shared and per-state
matrices, controlled gates with every control placement, cut phases) on random
n and pool sizes vs the oracle, bit for bit."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.graphs import make_graph
from oracle import gates as og, statevector as osv

def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.perf_counter()
fails = 0
for trial in range(trials):
    n = int(rng.integers(12, 17))
    S = int(rng.integers(1, 5))
    steps = int(rng.integers(20, 200))
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.2]
    graph = make_graph(n, edges)
    states = np.stack([og.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S)
    pool.state.upload(states)
    exp = states.copy()
    for _ in range(steps):
        r = rng.random()
        shared = rng.random() < 0.5
        if r < 0.55:
            q = int(rng.integers(n))
            us = np.stack([og.random_unitary_2x2(rng) for _ in range(1 if shared else S)])
            us = np.repeat(us, S, axis=0) if shared else us
            pool.queue.one_qubit(q, us[0] if shared else us)
            for s in range(S):
                osv.apply_1q(exp[s], q, us[s])
        elif r < 0.9:
            c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
            us = np.stack([og.random_unitary_2x2(rng) for _ in range(1 if shared else S)])
            if rng.random() < 0.3:
                us = np.stack([np.diag([1.0, np.exp(1j * rng.uniform(0, 6))]) for _ in range(len(us))])
            us = np.repeat(us, S, axis=0) if shared else us
            pool.queue.controlled(c, t, us[0] if shared else us)
            for s in range(S):
                osv.apply_controlled(exp[s], c, t, us[s])
        elif edges:
            g = rng.uniform(0, 6, size=S)
            pool.queue.cut_phase(graph, float(g[0]) if shared else g)
            for s in range(S):
                osv.apply_cut_phase(exp[s], edges, float(g[0] if shared else g[s]))
        if rng.random() < 0.05:
            pool.queue.flush()
    got = pool.amplitudes()
    if not bits_equal(got, exp):
        fails += 1
        print(f"trial {trial}: n={n} S={S} steps={steps} MISMATCH max|d|={np.abs(got - exp).max():.3e}")
print(f"{trials} trials, {fails} mismatches, {time.perf_counter() - t0:.1f} s")

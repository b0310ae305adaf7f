"""Randomised parity campaign for QS_FUSE_FACTORED: pool programs mixing
shared Haar / RX / RZ / X gates, per-state RX (factorable) and per-state Haar
(not), controlled gates with every control placement, CPhase and cut phases,
random flush points, on n=12..16 and pools of 1-4 states, vs the oracle to the
north_star tolerance (1e-12 on amplitudes; factored results are not bitwise).
  python tools/exp/fuzz_factored.py [trials] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import runtime  # noqa: E402
from paper_2001_10554_b200.graphs import make_graph  # noqa: E402
from oracle import gates as og, statevector as osv  # noqa: E402

X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
trials = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.perf_counter()
worst, fails = 0.0, 0
for trial in range(trials):
    n = int(rng.integers(12, 17))
    S = int(rng.integers(1, 5))
    steps = int(rng.integers(20, 200))
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.2]
    graph = make_graph(n, edges)
    states = np.stack([og.random_state(n, rng) for _ in range(S)])
    pool = runtime.PoolState(n, S, fuse="factored")
    pool.state.upload(states)
    exp = states.copy()
    for _ in range(steps):
        r = rng.random()
        q = int(rng.integers(n))
        if r < 0.5:
            kind = rng.random()
            if kind < 0.5:
                us = np.stack([og.random_unitary_2x2(rng)] * S)
            elif kind < 0.65:
                us = np.stack([og.rx(float(x)) for x in rng.uniform(0, 2 * np.pi, S)])
            elif kind < 0.75:
                us = np.stack([og.random_unitary_2x2(rng) for _ in range(S)])
            elif kind < 0.85:
                us = np.stack([og.rz(float(rng.uniform(0, 6.3)))] * S)
            else:
                us = np.stack([X] * S)
            shared = all(np.array_equal(us[0], u) for u in us)
            pool.queue.one_qubit(q, us[0] if shared else us)
            for s in range(S):
                osv.apply_1q(exp[s], q, us[s])
        elif r < 0.85:
            c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
            if rng.random() < 0.3:
                u = np.diag([1.0, np.exp(1j * rng.uniform(0, 6))]).astype(np.complex128)
            elif rng.random() < 0.5:
                u = X
            else:
                u = og.random_unitary_2x2(rng)
            pool.queue.controlled(c, t, u)
            for s in range(S):
                osv.apply_controlled(exp[s], c, t, u)
        elif edges:
            g = rng.uniform(0, 6, size=S)
            pool.queue.cut_phase(graph, g)
            for s in range(S):
                osv.apply_cut_phase(exp[s], edges, float(g[s]))
        if rng.random() < 0.03:
            pool.queue.flush()
    got = pool.amplitudes()
    dev = float(np.abs(got - exp).max())
    worst = max(worst, dev)
    if dev > 1e-12:
        fails += 1
        print(f"trial {trial}: n={n} S={S} steps={steps} max|d|={dev:.3e} > 1e-12")
print(f"{trials} trials, {fails} over 1e-12, worst max|d| {worst:.3e}, "
      f"{time.perf_counter() - t0:.1f} s")

"""Randomised parity campaign for the distributed paths: random circuits on
2/4/8 emulated ranks (global-qubit exchange, case (b)/(c)/(d) controlled
gates, cut phases) with and without qubit remapping, vs the oracle bit for bit."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.circuit import Circuit, GateSpec
from paper_2001_10554_b200.graphs import make_graph
from oracle import circuit as ocirc

def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
t0 = time.perf_counter()
fails = 0
for trial in range(trials):
    n = int(rng.integers(10, 15))
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.15]
    specs, plain = [], []
    for _ in range(int(rng.integers(20, 120))):
        r = rng.random()
        if r < 0.5:
            q = int(rng.integers(n))
            k = ("h", "x", "rx", "ry", "rz")[int(rng.integers(5))]
            th = float(rng.uniform(0, 6.28))
            specs.append(GateSpec(k, (q,), None if k in ("h", "x") else th))
            plain.append({"kind": k, "qubits": (q,), "param": th})
        elif r < 0.9:
            c, t = (int(x) for x in rng.choice(n, size=2, replace=False))
            k = ("cx", "cz")[int(rng.integers(2))]
            specs.append(GateSpec(k, (c, t)))
            plain.append({"kind": k, "qubits": (c, t)})
        elif edges:
            g = float(rng.uniform(0, 6.28))
            specs.append(GateSpec("diagcost", (), g, graph=make_graph(n, edges)))
            plain.append({"kind": "diagcost", "param": g, "edges": edges})
    circ = Circuit(n, tuple(specs))
    expected = ocirc.run(n, plain)
    for P in (2, 4, 8):
        for remap in (False, True):
            got = runtime.simulate_circuit(circ, num_ranks=P, remap=remap)
            if not bits_equal(got, expected):
                fails += 1
                print(f"trial {trial} n={n} P={P} remap={remap}: max|d|={np.abs(got - expected).max():.2e}")
print(f"{trials} circuits x 6 layouts, {fails} mismatches, {time.perf_counter() - t0:.1f} s")

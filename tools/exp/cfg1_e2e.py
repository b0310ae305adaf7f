"""Config 1 (n=20, 10 layers, 295 gates) through the public API: simulate_circuit
wall time per call (incl. the final state download) and the fused pass count."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import runtime
from paper_2001_10554_b200.circuit import Circuit
from paper_2001_10554_b200.workloads import config1_gates

n = 20
circ = Circuit(n, tuple(config1_gates(n, 10, 20260809)))
runtime.simulate_circuit(circ)  # warm-up (context, library)
for ranks in (1, 2, 4):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        psi = runtime.simulate_circuit(circ, num_ranks=ranks)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"config 1 (n=20, {len(circ.gates)} gates), {ranks} emulated rank(s): "
          f"median {ts[2] * 1e3:.1f} ms per simulate_circuit (incl. download of 2^20 amplitudes)")

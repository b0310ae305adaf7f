"""k_exchange_peer / k_swap_peer on one GPU: the "partner" is a second state on
the same device, so the timing is the kernel against HBM (the NVLink-bound
multi-GPU number cannot be taken here).  Each call moves 2^(m-1) amplitudes
each way (read + write both sides' halves: 64 B per pair)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200.workloads import haar_2x2

m = int(sys.argv[1]) if len(sys.argv) > 1 else 29
a = N.DeviceState(m + 1, m, 0, 1)
b = N.DeviceState(m + 1, m, 1, 1)
for st in (a, b):
    N.call("qs_init_gaussian", st.handle, 3)
u = haar_2x2(np.random.default_rng(0)).view(np.float64).ravel()
pb, pa = b.device_ptr(), a.device_ptr()
def run():
    N.call("qs_exchange_gate_peer", a.handle, pb, 1, N.dptr(u), -1)
    N.call("qs_exchange_gate_peer", b.handle, pa, 0, N.dptr(u), -1)
run(); a.synchronize(); b.synchronize()
ts = []
for _ in range(5):
    a.synchronize(); b.synchronize()
    t0 = time.perf_counter(); run(); a.synchronize(); b.synchronize()
    ts.append(time.perf_counter() - t0)
ms = np.median(ts) * 1e3
alg = 2 * 32 * 2 ** m  # both ranks' gate: 32 B per amplitude of each slice
print(f"exchange gate m={m}: {ms:.2f} ms for both ranks -> {alg / ms / 1e6:.0f} GB/s HBM "
      f"(algorithmic 32 B/amp per rank)")
for rb_q in ((m - 1, 0),):
    def swap():
        N.call("qs_swap_qubits_peer", a.handle, pb, rb_q[0], rb_q[1])
        N.call("qs_swap_qubits_peer", b.handle, pa, rb_q[0], rb_q[1])
    swap(); a.synchronize(); b.synchronize()
    t0 = time.perf_counter(); swap(); a.synchronize(); b.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    print(f"swap local {rb_q[0]} <-> rank bit: {ms:.2f} ms (each side moves 2^{m-1} amps)")

"""One launch of each secondary kernel at m=28 (ncu target): controlled gate,
cut phase, norm reduction, all-qubit marginals, exchange gate (partner on the
same GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200.workloads import haar_2x2

m = 28
st = N.DeviceState(m, m)
N.call("qs_init_gaussian", st.handle, 3)
u = haar_2x2(np.random.default_rng(0)).view(np.float64).ravel()
st.apply_program([N.QsGate(1, 20, 3, 0, 0, 0)], u, fuse=False)           # k_controlled
edges = np.array([(i, (i + 1) % 20) for i in range(20)], np.int32)
lut = np.exp(-1j * 0.3 * np.arange(21)).view(np.float64)
st.apply_program([N.QsGate(2, 0, -1, 0, 0, 0)], lut, edges, fuse=False)   # k_cut_phase
st.observable(0)                                                           # k_tree_wide (norm)
st.marginals()                                                             # k_marginals
b = N.DeviceState(m + 1, m, 1, 1)
a = N.DeviceState(m + 1, m, 0, 1)
N.call("qs_init_gaussian", a.handle, 4)
N.call("qs_init_gaussian", b.handle, 5)
N.call("qs_exchange_gate_peer", a.handle, b.device_ptr(), 1, N.dptr(u), -1)  # k_exchange_peer
st.synchronize(); a.synchronize()
print("ok")

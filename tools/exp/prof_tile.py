import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200.workloads import haar_2x2
lib = N.load()
m = int(sys.argv[1]); k = int(sys.argv[2])
st = N.DeviceState(m, m)
N.call("qs_init_gaussian", st.handle, 3)
rng = np.random.default_rng(1)
us = np.stack([haar_2x2(rng) for _ in range(k)]).view(np.float64).reshape(-1)
gates = [N.QsGate(0, i, -1, 0, 8 * i, 0) for i in range(k)]
st.apply_program(gates, us); st.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.qs_debug_prof(buf)
st.event_record(0); st.apply_program(gates, us); st.event_record(1)
ms = st.event_elapsed_ms(0, 1)
lib.qs_debug_prof(buf)
names = ["load+wait", "round LDS", "wait turn", "compute", "STS+gbar", "store"]
tot = sum(buf[:6])
print(f"m={m} gates={k} ms={ms:.3f}")
for i, n in enumerate(names):
    print(f"  {n:10s} {buf[i] / tot * 100:5.1f}%  per-warp-tile cycles {buf[i] / (1 << (m - 12)) / 8:.0f}")

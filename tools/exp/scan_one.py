import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200.workloads import haar_2x2
m = int(sys.argv[1]); k = int(sys.argv[2]); base = int(sys.argv[3]) if len(sys.argv) > 3 else 0
st = N.DeviceState(m, m)
N.call("qs_init_gaussian", st.handle, 3)
rng = np.random.default_rng(1)
us = np.stack([haar_2x2(rng) for _ in range(k)]).view(np.float64).reshape(-1)
gates = [N.QsGate(0, base + i, -1, 0, 8 * i, 0) for i in range(k)]
for _ in range(2):
    st.apply_program(gates, us, fuse=True)
st.synchronize()
print("ok")

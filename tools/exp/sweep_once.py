"""ncu target: the config-2 sweep program at m qubits, `reps` times.
  python tools/exp/sweep_once.py [m] [exact|factored] [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N  # noqa: E402
from paper_2001_10554_b200.workloads import haar_2x2  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
fuse = "factored" if (sys.argv[2] if len(sys.argv) > 2 else "factored") == "factored" else True
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
st = N.DeviceState(m, m)
N.call("qs_init_gaussian", st.handle, 3)
rng = np.random.default_rng(1)
for _ in range(reps):
    us = np.stack([haar_2x2(rng) for _ in range(m)]).view(np.float64).reshape(-1)
    st.apply_program([N.QsGate(0, q, -1, 0, 8 * q, 0) for q in range(m)], us, fuse=fuse)
st.synchronize()
print("ok")

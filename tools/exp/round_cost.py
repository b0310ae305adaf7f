"""One fused pass of k Haar gates on qubits base..base+k-1 (k <= 9 keeps one
pass), factored and exact: the per-round cost with HBM traffic.
  python tools/exp/round_cost.py [m] [base]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N  # noqa: E402
from paper_2001_10554_b200.workloads import haar_2x2  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
base = int(sys.argv[2]) if len(sys.argv) > 2 else 12
st = N.DeviceState(m, m)
N.call("qs_init_gaussian", st.handle, 3)
rng = np.random.default_rng(1)
for k in (1, 2, 4, 5, 8, 9):
    for mode in ("factored", True):
        us = np.stack([haar_2x2(rng) for _ in range(k)]).view(np.float64).reshape(-1)
        gates = [N.QsGate(0, base + i, -1, 0, 8 * i, 0) for i in range(k)]
        st.apply_program(gates, us, fuse=mode)
        ts = []
        for _ in range(5):
            st.event_record(0)
            passes = st.apply_program(gates, us, fuse=mode)
            st.event_record(1)
            st.synchronize()
            ts.append(st.event_elapsed_ms(0, 1))
        print(f"k={k} {'factored' if mode == 'factored' else 'exact':8s} passes={passes} "
              f"ms={np.median(ts):.3f}")

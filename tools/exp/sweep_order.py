"""Per-pass times of a factored config-2 sweep at n=M for several gate orders
(the list scheduler keeps program order when every gate needs a new tile
bit, so the order decides which qubits share a pass): how the number of
2 MiB pages a tile spans (tile bits >= 17) costs the TMA pass.
   M=30 python tools/exp/sweep_order.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N, runtime  # noqa: E402
from paper_2001_10554_b200.workloads import device_gaussian, haar_2x2  # noqa: E402

m = int(os.environ.get("M", "30"))
reps = int(os.environ.get("REPS", "5"))
R = list(range(m))
orders = {
    "natural": R,
    "reverse": R[::-1],
    "p2_6page": R[:12] + [12, 13, 14, 17, 18, 19, 20, 21, 22] + [15, 16] + R[23:],
    "p2_5page": R[:12] + [12, 13, 14, 15, 17, 18, 19, 20, 21] + [16] + R[22:],
    "p1_high": [0, 1, 2, 3, 4, 5, 6, 7, 26, 27, 28, 29] + R[8:26],
}
st = N.DeviceState(m, m)
device_gaussian(st, 5)
rng = np.random.default_rng(1)
q = runtime.GateQueue(st, fuse="factored")
for name, order in orders.items():
    assert sorted(order) == R, name

    def sweep():
        for k in order:
            q.one_qubit(k, haar_2x2(rng))
        q.flush()

    for _ in range(2):
        sweep()
    st.synchronize()
    st.launch_log(True)
    for _ in range(reps):
        sweep()
    st.synchronize()
    st.launch_log(False)
    ms, kinds = st.read_launch_log()
    per = ms.reshape(reps, -1).mean(axis=0)
    print(json.dumps({"order": name, "sweep_ms": round(float(per.sum()), 3),
                      "pass_ms": [round(float(x), 3) for x in per]}), flush=True)

"""One factored pass over tile {0,1,2} + qubits [lo, lo+8] (9 Haar gates) at
n=M: pass time vs the span of the tile's high bits (TLB / DRAM page study)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N, runtime  # noqa: E402
from paper_2001_10554_b200.workloads import device_gaussian, haar_2x2  # noqa: E402

m = int(os.environ.get("M", "30"))
reps = int(os.environ.get("REPS", "8"))
st = N.DeviceState(m, m)
device_gaussian(st, 5)
rng = np.random.default_rng(1)
q = runtime.GateQueue(st, fuse=os.environ.get("FUSE", "factored"))
out = {"tag": os.environ.get("TAG", "")}
for lo in [int(x) for x in os.environ.get("LOS", "3,12,15,17,19,21").split(",")]:
    def one():
        for k in range(lo, lo + 9):
            q.one_qubit(k, haar_2x2(rng))
        q.flush()
    one()
    st.synchronize()
    st.event_record(0)
    for _ in range(reps):
        one()
    st.event_record(1)
    st.synchronize()
    out[lo] = round(st.event_elapsed_ms(0, 1) / reps, 3)
print(json.dumps(out))

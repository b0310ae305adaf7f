"""Per-pass times of a config-4 layer at n=M (factored or exact)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N, runtime
from paper_2001_10554_b200.workloads import device_gaussian, haar_2x2
from paper_2001_10554_b200 import gates as G
m = int(os.environ.get("M", "30"))
fuse = os.environ.get("FUSE", "factored")
fuse = True if fuse == "exact" else fuse
reps = 5
st = N.DeviceState(m, m)
device_gaussian(st, 5)
rng = np.random.default_rng(1)
q = runtime.GateQueue(st, fuse=fuse)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
def layer():
    for k in range(m):
        q.one_qubit(k, haar_2x2(rng))
    for c in range(m // 2):
        q.controlled(c, m - 1 - c, X)
    q.flush()
for _ in range(2):
    layer()
st.synchronize(); st.launch_log(True); st.event_record(0)
for _ in range(reps):
    layer()
st.event_record(1); st.synchronize(); st.launch_log(False)
ms, kinds = st.read_launch_log()
total = st.event_elapsed_ms(0, 1) / reps
per = ms.reshape(reps, -1).mean(axis=0)
print(json.dumps({"m": m, "fuse": str(fuse), "layer_ms": round(total, 3),
                  "pass_ms": [round(float(x), 3) for x in per], "kinds": [int(k) for k in kinds[:len(per)]]}))

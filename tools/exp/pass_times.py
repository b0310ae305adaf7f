"""Per-pass times of the factored (or exact) config-2 sweep at n=M: launch
log (CUDA events per launch) over REPS sweeps after a warm-up.
   M=30 FUSE=factored REPS=10 python tools/exp/pass_times.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N, runtime  # noqa: E402
from paper_2001_10554_b200.workloads import device_gaussian, haar_2x2  # noqa: E402

m = int(os.environ.get("M", "30"))
fuse = os.environ.get("FUSE", "factored")
fuse = True if fuse == "exact" else fuse
reps = int(os.environ.get("REPS", "10"))
st = N.DeviceState(m, m)
device_gaussian(st, 5)
rng = np.random.default_rng(1)
q = runtime.GateQueue(st, fuse=fuse)


def sweep():
    for k in range(m):
        q.one_qubit(k, haar_2x2(rng))
    q.flush()


for _ in range(3):
    sweep()
st.synchronize()
st.launch_log(True)
st.event_record(0)
for _ in range(reps):
    sweep()
st.event_record(1)
st.synchronize()
st.launch_log(False)
ms, kinds = st.read_launch_log()
total = st.event_elapsed_ms(0, 1) / reps
per = ms.reshape(reps, -1).mean(axis=0)
tag = os.environ.get("TAG", "")
print(json.dumps({"tag": tag, "m": m, "fuse": str(fuse), "sweep_ms": round(total, 3),
                  "pass_ms": [round(float(x), 3) for x in per], "kinds": [int(k) for k in kinds[:len(per)]]}))

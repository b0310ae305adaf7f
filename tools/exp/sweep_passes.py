"""Per-pass times of the config-2 sweep (30 Haar gates at m qubits) from the
library's launch log, for each fuse mode given:
  python tools/exp/sweep_passes.py [m] [exact|factored ...]
QSB_LIB=<variant .so> times a tools/exp/variants build instead."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2001_10554_b200 import _native as N  # noqa: E402
from paper_2001_10554_b200.workloads import haar_2x2  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
modes = sys.argv[2:] or ["exact", "factored"]
st = N.DeviceState(m, m)
N.call("qs_init_gaussian", st.handle, 3)
rng = np.random.default_rng(1)
for mode in modes:
    fuse = "factored" if mode == "factored" else True
    rows = []
    for rep in range(6):
        us = np.stack([haar_2x2(rng) for _ in range(m)]).view(np.float64).reshape(-1)
        gates = [N.QsGate(0, q, -1, 0, 8 * q, 0) for q in range(m)]
        st.launch_log(rep > 0)
        st.event_record(0)
        st.apply_program(gates, us, fuse=fuse)
        st.event_record(1)
        st.synchronize()
        if rep > 0:
            ms, kinds = st.read_launch_log()
            rows.append((st.event_elapsed_ms(0, 1), list(np.round(ms, 3))))
        st.launch_log(False)
    tot = np.median([r[0] for r in rows])
    per = np.median(np.array([r[1] for r in rows]), axis=0)
    print(f"{mode}: sweep {tot:.2f} ms, passes {list(np.round(per, 3))}")

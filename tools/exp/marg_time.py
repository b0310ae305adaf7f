import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import _native as N
m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
st = N.DeviceState(m, m, 0, S)
N.call("qs_init_gaussian", st.handle, 3)
st.marginals(); st.synchronize()
for name, fn in (("marginals", lambda: st.marginals()), ("norm", lambda: st.observable(0)),
                 ("prob q=5", lambda: st.observable(1, 5))):
    t = []
    for _ in range(5):
        st.synchronize(); t0 = time.perf_counter(); fn(); t.append(time.perf_counter() - t0)
    ms = np.median(t) * 1e3
    print(f"m={m} S={S} {name}: {ms:.2f} ms  ({16 * 2**m * S / ms / 1e6:.0f} GB/s read)")

"""qs_exchange_gate_nccl through a single-rank communicator (self-exchange) at
m=29: the pipeline's cost against HBM (send/recv are device-local copies here;
across GPUs the same bytes cross NVLink)."""
import ctypes, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200.workloads import haar_2x2

m = int(sys.argv[1]) if len(sys.argv) > 1 else 29
st = N.DeviceState(m + 1, m, 0, 1, 0)
N.call("qs_init_gaussian", st.handle, 3)
uid = (ctypes.c_ubyte * 128)()
N.call("qs_nccl_unique_id", uid)
N.call("qs_comm_init", st.handle, uid, 1, 0)
u = haar_2x2(np.random.default_rng(0)).view(np.float64).ravel()
for chunk_log2 in (22, 24, 26):
    f = lambda: N.call("qs_exchange_gate_nccl", st.handle, 0, 1, N.dptr(u), -1, 1 << chunk_log2)
    f()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    ms = np.median(ts) * 1e3
    print(f"m={m} chunk 2^{chunk_log2}: {ms:.2f} ms per exchange gate "
          f"({2 ** m * 16 / ms / 1e6:.0f} GB/s of slice sent+received)")
N.call("qs_comm_destroy", st.handle)

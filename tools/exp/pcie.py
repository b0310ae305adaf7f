"""PCIe probe: pinned upload / download / full-duplex exchange of a 2^m state."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2001_10554_b200 import _native as N  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = N.DeviceState(m, m, 0, 1, 0)
a = torch.empty(2 << m, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
b = torch.empty(2 << m, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
a[:] = 1.0
GB = 16 * (1 << m) / 1e9
for rep in range(2):
    t = time.perf_counter(); st.upload(a); st.synchronize(); up = time.perf_counter() - t
    t = time.perf_counter(); st.download(b); dn = time.perf_counter() - t
    print(f"upload {GB / up:.1f} GB/s  download {GB / dn:.1f} GB/s")
for chunk in (1 << 20, 1 << 22, 1 << 24, 1 << 26):
    t = time.perf_counter(); st.exchange_host(a, b, chunk); ex = time.perf_counter() - t
    print(f"exchange chunk 2^{chunk.bit_length() - 1}: {ex * 1e3:.0f} ms  {GB / ex:.1f} GB/s each way")

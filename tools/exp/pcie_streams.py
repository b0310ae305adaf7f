"""Full-duplex PCIe with 1 or 2 streams per direction (torch copies)."""
import time
import torch

n = 1 << 30  # 2^30 complex128 = 16 GiB per direction
host_in = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
host_out = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
dev = torch.empty(2 * n, dtype=torch.float64, device="cuda")
host_in.fill_(1.0)
GB = 16 * n / 1e9
chunk = 2 * (1 << 24)
for per_dir in (1, 2, 4):
    up = [torch.cuda.Stream() for _ in range(per_dir)]
    dn = [torch.cuda.Stream() for _ in range(per_dir)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, off in enumerate(range(0, 2 * n, chunk)):
            s_dn, s_up = dn[i % per_dir], up[i % per_dir]
            with torch.cuda.stream(s_dn):
                host_out[off:off + chunk].copy_(dev[off:off + chunk], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_dn)
            s_up.wait_event(ev)
            with torch.cuda.stream(s_up):
                dev[off:off + chunk].copy_(host_in[off:off + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{per_dir} stream(s)/direction: {dt * 1e3:.0f} ms, {GB / dt:.1f} GB/s each way")

"""Cost of pinning caller memory in place (cudaHostRegister) vs staging copies,
for the pageable e2e path.  python tools/host_register_probe.py"""
import time

import numpy as np
import torch

cr = torch.cuda.cudart()
n = 256 << 20
for trial in range(3):
    a = np.random.default_rng(trial).integers(0, 256, n, dtype=np.uint8)   # fresh pageable buffer
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(a.ctypes.data, n, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print(f"256 MiB: register {1e3 * (t1 - t0):.1f} ms (rc {rc}), H2D {n / (t2 - t1) / 1e9:.1f} GB/s, "
          f"unregister {1e3 * (t3 - t2):.1f} ms")

"""Host copy bandwidth of the pageable -> pinned staging step (numpy copyto on
N threads, GIL released), the bound on the pageable-input e2e path.

    python tools/host_copy_bw.py
"""
import concurrent.futures as cf
import os
import time

import numpy as np
import torch

N = 256 << 20
src = np.random.default_rng(0).integers(0, 256, N, dtype=np.uint8)
dst_pin = torch.empty(N, dtype=torch.uint8, pin_memory=True).numpy()
dst_page = np.empty(N, dtype=np.uint8)
dst_page[:] = 1
print("cpus", os.cpu_count())
for name, dst in (("pinned", dst_pin), ("pageable", dst_page)):
    for threads in (1, 2, 4, 8, 16, 32):
        if threads > 2 * (os.cpu_count() or 1):
            continue
        pool = cf.ThreadPoolExecutor(threads)
        edges = [N * i // threads for i in range(threads + 1)]
        def one(i):
            np.copyto(dst[edges[i]:edges[i + 1]], src[edges[i]:edges[i + 1]])
        list(pool.map(one, range(threads)))
        t = time.perf_counter()
        for _ in range(5):
            list(pool.map(one, range(threads)))
        dt = (time.perf_counter() - t) / 5
        print(f"{name:9s} threads={threads:2d}: {N / dt / 1e9:6.1f} GB/s")
        pool.shutdown()

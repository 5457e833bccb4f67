"""Host<->device copy bandwidth on this box (pinned and pageable), for the e2e roofline."""
import time

import torch

n = 256 << 20
for pinned in (True, False):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=pinned)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=pinned)
    torch.cuda.synchronize()
    h2d = 5 * n / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    for _ in range(5):
        h.copy_(d, non_blocking=pinned)
    torch.cuda.synchronize()
    d2h = 5 * n / (time.perf_counter() - t) / 1e9
    print(f"{'pinned' if pinned else 'pageable'}: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s")

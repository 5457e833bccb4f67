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

# two 256 MiB pinned copies on two streams at once (the e2e path's x / y legs),
# and the same split into 64 MiB chunks
hx = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(1)
hy = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(2)
dx = torch.empty(n, dtype=torch.uint8, device="cuda")
dy = torch.empty(n, dtype=torch.uint8, device="cuda")
sx, sy = torch.cuda.Stream(), torch.cuda.Stream()
for chunk in (n, 64 << 20, 16 << 20):
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for lo in range(0, n, chunk):
            with torch.cuda.stream(sx):
                dx[lo:lo + chunk].copy_(hx[lo:lo + chunk], non_blocking=True)
            with torch.cuda.stream(sy):
                dy[lo:lo + chunk].copy_(hy[lo:lo + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"pinned x+y on two streams, {chunk >> 20} MiB chunks: {2 * n / dt / 1e9:.1f} GB/s")

# the same 2 x 256 MiB over 4 streams (each operand split in halves)
ss = [torch.cuda.Stream() for _ in range(4)]
half = n // 2
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i, (d, h) in enumerate(((dx, hx), (dy, hy))):
        for j in range(2):
            with torch.cuda.stream(ss[2 * i + j]):
                d[j * half:(j + 1) * half].copy_(h[j * half:(j + 1) * half], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"pinned x+y on four streams: {2 * n / dt / 1e9:.1f} GB/s")

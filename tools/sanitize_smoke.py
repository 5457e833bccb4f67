"""Small run of every kernel family for compute-sanitizer (one tool per call).

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import pathlib
import random
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from oracle import coracle
from paper_2402_14607_b200 import _lib
from paper_2402_14607_b200 import device as D
from paper_2402_14607_b200 import workloads as W

rnd = random.Random(3)
fails = 0
cases = [(4, 64, 700, 0), (2, 64, 300, 0), (8, 64, 129, 0), (16, 64, 77, 0), (32, 64, 40, 0),
         (64, 8, 55, 0), (128, 8, 33, 0), (56, 48, 45, 3), (58, 120, 17, 5), (80, 71, 9, 0),
         (13, 7, 300, 11), (1, 24, 500, 1), (3, 50, 90, 0), (127, 3, 40, 9), (100, 2000, 3, 0),
         (56, 48, 45, 0), (24, 16, 70, 0), (40, 32, 33, 0), (48, 8, 65, 0)]   # period kernel
for q, n, k, off in cases:
    nb = (off + k * q * n + 7) // 8
    xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
    xd, xn = D.to_device_stream(xb, "cuda")
    yd, yn = D.to_device_stream(yb, "cuda")
    for oo in (0, 5):
        out = D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=off, y_bit0=off, out_bit0=oo)
        got = int.from_bytes(out.cpu().numpy().tobytes(), "little") >> oo
        want = int.from_bytes(coracle.extract_eq(xb, yb, q, n, k, x_bit0=off, y_bit0=off), "little")
        ok = (got & ((1 << (k * q)) - 1)) == want
        fails += not ok
        print(q, n, k, off, oo, _lib.launch_info(q, n, k)["family"], "ok" if ok else "MISMATCH")
# neq, pack, sources
xd, xn = D.to_device_stream(rnd.randbytes(4000), "cuda")
D.extract_neq(xd, xn, xd, xn, 8, 8, 5, 6)
D.pack(torch.arange(1000, device="cuda", dtype=torch.int16), 11, out_bit0=3)
D.bernoulli_bits(10_000, 0.2, 5, bit0=512)
m = D.empty_stream(64 * 1000, "cuda")
m[:64000] = 1
D.xor_scan_rows(m, 1000, 64)
u = torch.rand(5000, dtype=torch.float64, device="cuda")
t = np.random.default_rng(1).random((16, 16))
cum = np.cumsum(t / t.sum(1, keepdims=True), axis=1)
cum[:, -1] = 1.0
D.markov_chain(u, torch.from_numpy(cum).cuda(), 4, 3)
# neq with growing widths and random run shapes on the TMA / staged / direct paths
for _ in range(40):
    q = rnd.randint(1, 128)
    n = rnd.randint(1, 90)
    k = rnd.randint(1, 600)
    xo, yo, oo = rnd.randint(0, 200), rnd.randint(0, 200), rnd.randint(0, 70)
    nb = (max(xo, yo) + k * q * n + 7) // 8
    xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
    xd, xn = D.to_device_stream(xb, "cuda")
    yd, yn = D.to_device_stream(yb, "cuda")
    D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=xo, y_bit0=yo, out_bit0=oo)
torch.cuda.synchronize()
viol, first = _lib.checked_violations()
print("fails", fails, "checked_violations", viol, "first", first)
sys.exit(1 if fails or viol > 0 else 0)

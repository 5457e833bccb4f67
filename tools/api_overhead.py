"""Where the fixed cost of a small extract_eq(...).run() goes (config 1 shape:
2^20 bits per source, q=32, n=4 -> 8192 blocks).  Median microseconds of 300
calls after warm-up for each piece of the call, on cuda:0."""
import io
import json
import statistics
import sys
import time
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import paper_2402_14607_b200 as bx  # noqa: E402
from paper_2402_14607_b200 import device as D, sharding  # noqa: E402


def med(fn, n=300):
    for _ in range(30):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


def main():
    q, n, k = 32, 4, 8192
    B = q * n
    rng = np.random.default_rng(1)
    x1 = rng.integers(0, 256, k * B // 8, dtype=np.uint8).tobytes()
    y1 = rng.integers(0, 256, k * B // 8, dtype=np.uint8).tobytes()
    plan = bx.EqPlan(1, k * B, Fraction(1), Fraction(1, 2), n, q, k, k * q, 0.0)
    xd, xn = D.to_device_stream(x1, "cuda")
    yd, yn = D.to_device_stream(y1, "cuda")
    out = torch.zeros(D.padded_len(k * q // 8), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    hp = torch.empty(len(x1), dtype=torch.uint8, pin_memory=True)
    res = {}
    res["launch_only_no_sync"] = med(lambda: D.extract_eq(xd, xn, yd, yn, q, n, k, out=out, stream=st))
    torch.cuda.synchronize()
    res["launch_plus_sync"] = med(lambda: (D.extract_eq(xd, xn, yd, yn, q, n, k, out=out, stream=st),
                                           st.synchronize()))
    res["h2d_128KiB_pinned_sync"] = med(lambda: (xd[:xn].copy_(hp, non_blocking=True), st.synchronize()))
    res["zero_plus_sync"] = med(lambda: (out.zero_(), st.synchronize()))
    from paper_2402_14607_b200 import _lib
    L = _lib.lib()
    xa = np.frombuffer(x1, np.uint8)
    ya = np.frombuffer(y1, np.uint8)
    oa = np.empty(k * q // 8, np.uint8)
    res["c_host_call"] = med(lambda: L.bx_extract_eq_host(xa.ctypes.data, xa.size, 0, ya.ctypes.data,
                                                          ya.size, 0, q, n, k, oa.ctypes.data, 0))
    xq, yq = x1[:4096 * 4], y1[:4096 * 4]          # 1/8 of the bytes: the copy share
    res["c_host_call_eighth"] = med(lambda: L.bx_extract_eq_host(
        np.frombuffer(xq, np.uint8).ctypes.data, len(xq), 0, np.frombuffer(yq, np.uint8).ctypes.data,
        len(yq), 0, q, n, k // 8, oa.ctypes.data, 0))
    res["extract_packed"] = med(lambda: sharding.extract_packed(x1, y1, q, n, k))
    f32, f128 = bx.field(32), bx.field(128)
    res["gf_mul_q32"] = med(lambda: f32.mul(0x12345678, 0x9ABCDEF1), 200)
    res["gf_mul_q128"] = med(lambda: f128.mul((1 << 127) | 12345, (1 << 100) | 777), 200)
    res["gf_inv_q128"] = med(lambda: f128.inv((1 << 127) | 12345), 100)
    xs = [list(range(1, 72))] * 64
    f80 = bx.field(80)
    pairs = [bx.BlockPair(i + 1, f80, tuple(v), tuple(reversed(v))) for i, v in enumerate(xs)]
    res["run_parallel_64_blocks_q80_n71"] = med(lambda: list(bx.run_parallel(iter(pairs), 1)), 50)
    res["api_run"] = med(lambda: bx.extract_eq(x1, y1, plan).run(io.BytesIO()))
    print(json.dumps(res))


if __name__ == "__main__":
    main()

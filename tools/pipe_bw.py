"""Throughput of the native streaming pipe (bx_pipe) and
the fixed cost of one small extract_eq(...).run() call (config 1).

    python tools/pipe_bw.py [--mb 512] [--chunk-mb 16]

Pipe: two seeded host streams of --mb MiB each pushed in --chunk-mb pieces
(pageable host memory, as a capture loop would hand them over) through
Pipe(depth=1) (synchronous) and Pipe(depth=2) (push k+1's host copy and H2D
overlap push k's kernel and D2H); raw input Gbit/s = 2 * 8 * bytes / time.
The outputs are compared with one device run over the same streams.
API: extract_eq(x, y, plan).run(sink) on config 1's shape (2^20 bits per
source, q=32, n=4 -> 8192 blocks), median of 200 calls after warm-up.
"""
import argparse
import io
import json
import statistics
import sys
import time
from fractions import Fraction

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))

import torch  # noqa: E402

import paper_2402_14607_b200 as bx  # noqa: E402
from paper_2402_14607_b200 import device as D  # noqa: E402
from paper_2402_14607_b200.pipe import Pipe  # noqa: E402


def pipe_rate(xb, yb, q, n, chunk, depth, reps=3):
    """Best of `reps` runs over pre-cut chunks (a capture loop's buffers);
    the pipe is created outside the timing (its pinned buffers are set up once)."""
    xs = [memoryview(xb)[pos:pos + chunk] for pos in range(0, len(xb), chunk)]
    ys = [memoryview(yb)[pos:pos + chunk] for pos in range(0, len(yb), chunk)]
    best = None
    for _ in range(reps):
        out = []
        with Pipe(q, n, chunk_bytes=chunk, depth=depth) as p:
            t0 = time.perf_counter()
            for a, b in zip(xs, ys):
                out.append(p.push(a, b))
            out.append(p.flush())
            dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return 2 * 8 * len(xb) / best / 1e9, b"".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=512)
    ap.add_argument("--chunk-mb", type=int, default=16)
    args = ap.parse_args()
    res = {}
    rng = np.random.default_rng(3)
    nbytes = args.mb << 20
    xb = rng.integers(0, 256, nbytes, dtype=np.uint8).tobytes()
    yb = rng.integers(0, 256, nbytes, dtype=np.uint8).tobytes()
    res["host_copy_threads"] = int(__import__("os").environ.get("BX_PIPE_THREADS", "4")) + 1
    for q, n in ((4, 64), (16, 64)):
        k = nbytes * 8 // (q * n)
        xd, xn = D.to_device_stream(xb, "cuda")
        yd, yn = D.to_device_stream(yb, "cuda")
        want = D.extract_eq(xd, xn, yd, yn, q, n, k)[:(k * q + 7) // 8].cpu().numpy().tobytes()
        del xd, yd
        for depth in (1, 2, 3):
            pipe_rate(xb[:args.chunk_mb << 21], yb[:args.chunk_mb << 21], q, n,
                      args.chunk_mb << 20, depth, reps=1)      # warm-up
            g, got = pipe_rate(xb, yb, q, n, args.chunk_mb << 20, depth)
            res[f"pipe_q{q}_n{n}_depth{depth}"] = {"raw_gbps": g, "bit_exact": got == want}
    # fixed cost of a small API call (config 1 shape)
    q, n, k = 32, 4, 8192
    B = q * n
    x1 = rng.integers(0, 256, k * B // 8, dtype=np.uint8).tobytes()
    y1 = rng.integers(0, 256, k * B // 8, dtype=np.uint8).tobytes()
    plan = bx.EqPlan(1, k * B, Fraction(1), Fraction(1, 2), n, q, k, k * q, 0.0)
    for _ in range(20):
        bx.extract_eq(x1, y1, plan).run(io.BytesIO())
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        bx.extract_eq(x1, y1, plan).run(io.BytesIO())
        ts.append(time.perf_counter() - t0)
    res["api_c1_call_us"] = {"median": statistics.median(ts) * 1e6, "min": min(ts) * 1e6,
                             "raw_gbps_median": 2 * k * B / statistics.median(ts) / 1e9}
    print(json.dumps(res))


if __name__ == "__main__":
    main()

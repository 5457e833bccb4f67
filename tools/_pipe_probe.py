import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2402_14607_b200.pipe import Pipe
from paper_2402_14607_b200 import _lib
rng = np.random.default_rng(1)
chunk = 16 << 20
xb = rng.integers(0, 256, 8 * chunk, dtype=np.uint8).tobytes()
yb = rng.integers(0, 256, 8 * chunk, dtype=np.uint8).tobytes()
xs = [xb[i*chunk:(i+1)*chunk] for i in range(8)]
ys = [yb[i*chunk:(i+1)*chunk] for i in range(8)]
for q, n in ((4, 64), (16, 64)):
    for depth in (1, 2):
        for rep in range(2):
            t0 = time.perf_counter()
            p = Pipe(q, n, chunk_bytes=chunk, depth=depth)
            t1 = time.perf_counter()
            ts = []
            for i in range(8):
                a = time.perf_counter(); p.push(xs[i], ys[i]); ts.append((time.perf_counter() - a) * 1e3)
            a = time.perf_counter(); p.flush(); tf = (time.perf_counter() - a) * 1e3
            p.close()
            print(q, depth, rep, 'create %.1f ms' % ((t1 - t0) * 1e3), 'push ms', ['%.2f' % t for t in ts], 'flush %.2f' % tf, flush=True)

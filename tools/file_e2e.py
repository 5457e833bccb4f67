"""File-object inputs through the public API (the README / CLI usage):
extract_eq(open(x), open(y), plan).run(open(out, "wb")) on two 256 MiB files.

    python tools/file_e2e.py
"""
import pathlib
import sys
import tempfile
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np

import paper_2402_14607_b200 as bx

d = pathlib.Path(tempfile.mkdtemp())
r = np.random.default_rng(0)
(d / "x.bin").write_bytes(r.integers(0, 256, 2**28, dtype=np.uint8).tobytes())
(d / "y.bin").write_bytes(r.integers(0, 256, 2**28, dtype=np.uint8).tobytes())
plan = bx.plan_eq(8, 2**28, "3/4", "2^-30")
for i in range(4):
    t = time.perf_counter()
    with open(d / "x.bin", "rb") as fx, open(d / "y.bin", "rb") as fy, open(d / "o.bin", "wb") as fo:
        rep = bx.extract_eq(fx, fy, plan).run(fo)
    dt = time.perf_counter() - t
    print(f"file -> file (page cache): {dt * 1e3:.0f} ms, {2 * 2**28 * 8 / dt / 1e9:.1f} Gbit/s raw in, "
          f"{rep.blocks_completed} blocks")

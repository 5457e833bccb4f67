"""Profile the end-to-end public-API path (host time breakdown) on a GPU box.

    python tools/e2e_probe.py --workload c3
"""
import argparse
import cProfile
import io
import pathlib
import pstats
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--sink", default="bytesio", choices=["bytesio", "null", "keep"])
a = ap.parse_args()
wl = W.WORKLOADS[a.workload]
nb = wl.stream_bytes
x = torch.randint(0, 256, (nb,), dtype=torch.uint8).pin_memory()
y = torch.randint(0, 256, (nb,), dtype=torch.uint8).pin_memory()
plan = wl.plan()


class Null:
    def write(self, b):
        return len(b)


class Keep:
    def write(self, b):
        self.data = b
        return len(b)


mk = {"bytesio": io.BytesIO, "null": Null, "keep": Keep}[a.sink]
bx.extract_eq(x, y, plan).run(mk())
torch.cuda.synchronize()
for _ in range(2):
    t = time.perf_counter()
    bx.extract_eq(x, y, plan).run(mk())
    torch.cuda.synchronize()
    print(f"{a.workload} sink={a.sink}: {(time.perf_counter() - t) * 1e3:.1f} ms, "
          f"{2 * wl.block_bits * wl.num_blocks / (time.perf_counter() - t) / 1e9:.1f} Gbit/s")
pr = cProfile.Profile()
pr.enable()
bx.extract_eq(x, y, plan).run(mk())
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(12)
print(s.getvalue()[:3000])

"""Pageable-input e2e for a few staging settings (run once per setting)."""
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200 import workloads as W


class Keep:
    def write(self, b):
        self.b = b


wl = W.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
x = np.random.default_rng(0).integers(0, 256, wl.stream_bytes, dtype=np.uint8).tobytes()
y = np.random.default_rng(1).integers(0, 256, wl.stream_bytes, dtype=np.uint8).tobytes()
plan = wl.plan()
bx.extract_eq(x, y, plan).run(Keep())
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    bx.extract_eq(x, y, plan).run(Keep())
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"{wl.name}: {2 * wl.block_bits * wl.num_blocks / dt / 1e9:.1f} Gbit/s pageable e2e")

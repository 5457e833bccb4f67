"""Minimal driver for profiling one extraction kernel under ncu.

    python tools/prof_eq.py --workload c2 --launches 3

Device-resident random streams of the workload's size (torch RNG; contents do
not matter for timing), then `--launches` bx_extract_eq calls.  Prints the
mean event-timed duration (not valid under ncu)."""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch

from paper_2402_14607_b200 import _lib
from paper_2402_14607_b200 import device as D
from paper_2402_14607_b200 import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--q", type=int)
    ap.add_argument("--n", type=int)
    ap.add_argument("--blocks", type=int)
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--real", action="store_true", help="the workload's seeded streams instead of random bytes")
    a = ap.parse_args()
    wl = W.WORKLOADS[a.workload]
    q, n = a.q or wl.q, a.n or wl.n
    nblocks = a.blocks or wl.num_blocks
    nbytes = (nblocks * q * n + 7) // 8
    g = torch.Generator(device="cuda").manual_seed(0)
    if a.real:
        x, _ = W.stream_device(wl.x, wl.samples, torch.device("cuda"))
        y, _ = W.stream_device(wl.y, wl.samples, torch.device("cuda"))
    else:
        x = D.empty_stream(nbytes, "cuda")
        y = D.empty_stream(nbytes, "cuda")
        x[:nbytes] = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda", generator=g)
        y[:nbytes] = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.zeros(D.padded_len((nblocks * q + 7) // 8), dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    D.extract_eq(x, nbytes, y, nbytes, q, n, nblocks, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.launches):
        D.extract_eq(x, nbytes, y, nbytes, q, n, nblocks, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.launches
    gbs = nblocks * (2 * q * n / 8 + q / 8) / (ms * 1e-3) / 1e9
    print(f"q={q} n={n} blocks={nblocks}: {ms:.4f} ms/launch, {gbs:.1f} GB/s algorithmic, "
          f"{2 * q * n * nblocks / (ms * 1e-3) / 1e9:.1f} Gbit/s raw in; "
          f"{_lib.launch_info(q, n, nblocks)}")


if __name__ == "__main__":
    main()

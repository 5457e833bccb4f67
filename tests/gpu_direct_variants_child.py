"""Child process of test_gpu_direct_variants: parity of the aligned one-thread-
per-block kernels (eq_direct_kernel for powers of two, eq_period_kernel for
q = 24, 40, 48, 56) under the load-width knob in the environment (BX_WIDE is
read once per process).
Prints 'ok <cases>' or raises."""
import math
import os
import pathlib
import random
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch

from oracle import coracle
from paper_2402_14607_b200 import _lib, device as D


def main():
    rnd = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
    cases = 0
    for q in (1, 2, 4, 8, 16, 32, 64, 128, 24, 40, 48, 56):
        period = q // math.gcd(q, 128)        # 128-bit units per element period
        for units in (1, 2, 3, 4, 5, 8, 9, 16, period, 2 * period, 3 * period):
            if (128 * units) % q:
                continue
            n = 128 * units // q
            for k in (1, 7, 33, rnd.randint(100, 3000)):
                oo = rnd.choice([0, 32, 96])
                nb = k * q * n // 8
                xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
                xd, _ = D.to_device_stream(xb, "cuda")
                yd, _ = D.to_device_stream(yb, "cuda")
                obytes = (oo + k * q + 7) // 8
                out = torch.full((D.padded_len(obytes),), 0xA5, dtype=torch.uint8, device="cuda")
                D.extract_eq(xd, nb, yd, nb, q, n, k, out=out, out_bit0=oo)
                got = int.from_bytes(out[:obytes].cpu().numpy().tobytes(), "little")
                want = int.from_bytes(coracle.extract_eq(xb, yb, q, n, k), "little")
                assert (got >> oo) & ((1 << (k * q)) - 1) == want, (q, n, k, oo)
                pre = int.from_bytes(bytes([0xA5]) * obytes, "little")
                keep = ((1 << obytes * 8) - 1) ^ (((1 << (k * q)) - 1) << oo)
                assert got & keep == pre & keep, ("canary", q, n, k, oo)
                assert _lib.launch_info(q, n, k)["direct"], (q, n)
                cases += 1
    if os.environ.get("BX_LIB") == "checked":
        n, first = _lib.checked_violations()
        assert n == 0, ("bounds violations", n, first)
    print("ok", cases)


if __name__ == "__main__":
    main()

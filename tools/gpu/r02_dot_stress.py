"""One-off randomized stress of the dot-product (IDP.2A) kernels against the C
oracle: every q in 9..64 (tile kernels, all thread splits, bit offsets), the
direct q = 16 / 32 kernels and the period widths, several seeds, plus dense
(all-ones / high-weight) inputs that maximise the per-field counts.

    python tools/gpu/r02_dot_stress.py [seeds]   ->  'ok <cases>'"""
import pathlib
import random
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))

import numpy as np
import torch

from oracle import coracle
from paper_2402_14607_b200 import device as D


def run(xb, yb, q, n, k, xo=0, yo=0):
    xd, xn = D.to_device_stream(xb, "cuda")
    yd, yn = D.to_device_stream(yb, "cuda")
    nbytes = (k * q + 7) // 8
    out = torch.zeros(D.padded_len(nbytes), dtype=torch.uint8, device="cuda")
    D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=xo, y_bit0=yo, out=out)
    return out[:nbytes].cpu().numpy().tobytes()


def dense(rnd, nb, p):
    """bytes with bit density p (p = 1: all ones)"""
    if p >= 1:
        return b"\xff" * nb
    bits = np.frombuffer(rnd.randbytes(nb * 8), dtype=np.uint8) < int(256 * p)
    return np.packbits(bits, bitorder="little").tobytes()


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cases = 0
    for seed in range(seeds):
        rnd = random.Random(1000 + seed)
        for q in range(9, 65):
            for n in (rnd.randint(4, 15), rnd.randint(16, 63), rnd.choice([64, 71, 120, 128]),
                      rnd.randint(129, 400)):
                k = rnd.randint(1, 300)
                xo, yo = rnd.choice([(0, 0), (rnd.randint(0, 63), rnd.randint(0, 63))])
                nb = (max(xo, yo) + k * q * n + 7) // 8 + 4
                p = rnd.choice([0.5, 0.5, 0.9, 1.0])
                xb, yb = dense(rnd, nb, p), dense(rnd, nb, rnd.choice([0.5, 1.0]))
                want = coracle.extract_eq(xb, yb, q, n, k, x_bit0=xo, y_bit0=yo)
                assert run(xb, yb, q, n, k, xo, yo) == want, (seed, q, n, k, xo, yo, p)
                cases += 1
        # aligned direct / period shapes at sizes that fill many CTAs
        for q, n in ((16, 64), (16, 8), (32, 64), (32, 4), (32, 12), (24, 64), (40, 48), (48, 64),
                     (56, 48), (56, 16), (64, 50), (64, 64)):
            k = rnd.randint(20000, 60000)
            nb = k * q * n // 8
            p = rnd.choice([0.5, 0.95, 1.0])
            xb, yb = dense(rnd, nb, p), dense(rnd, nb, p)
            assert run(xb, yb, q, n, k) == coracle.extract_eq(xb, yb, q, n, k), (seed, q, n, k, p)
            cases += 1
    print("ok", cases)


if __name__ == "__main__":
    main()

"""One-off randomized stress of every kernel family against the C oracle on the
final round-2 tree: every q in 1..128, random vector lengths, block counts and
bit offsets (aligned shapes hit the direct / period kernels, the rest the TMA /
staged kernels), uniform and dense inputs.

    python tools/gpu/r02_all_q_stress.py [seeds]   ->  'ok <cases>'"""
import pathlib
import random
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))

import torch

from oracle import coracle
from paper_2402_14607_b200 import device as D


def run(xb, yb, q, n, k, xo, yo, oo):
    xd, xn = D.to_device_stream(xb, "cuda")
    yd, yn = D.to_device_stream(yb, "cuda")
    nbytes = (oo + k * q + 7) // 8
    out = torch.zeros(D.padded_len(nbytes), dtype=torch.uint8, device="cuda")
    D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=xo, y_bit0=yo, out=out, out_bit0=oo)
    return int.from_bytes(out[:nbytes].cpu().numpy().tobytes(), "little") >> oo


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cases = 0
    for seed in range(seeds):
        rnd = random.Random(7000 + seed)
        for q in range(1, 129):
            for _ in range(3):
                n = rnd.choice([rnd.randint(1, 12), rnd.randint(13, 80), rnd.choice([32, 64, 128, 256]),
                                rnd.randint(81, 500)])
                k = rnd.randint(1, 400)
                aligned = rnd.random() < 0.4
                xo, yo = (0, 0) if aligned else (rnd.randint(0, 200), rnd.randint(0, 200))
                oo = 0 if aligned else rnd.choice([0, rnd.randint(1, 70)])
                nb = (max(xo, yo) + k * q * n + 7) // 8 + rnd.randint(0, 5)
                fill = rnd.choice([None, None, b"\xff"])
                xb = fill * nb if fill else rnd.randbytes(nb)
                yb = rnd.randbytes(nb) if rnd.random() < 0.8 else b"\xff" * nb
                want = int.from_bytes(coracle.extract_eq(xb, yb, q, n, k, x_bit0=xo, y_bit0=yo), "little")
                got = run(xb, yb, q, n, k, xo, yo, oo) & ((1 << (k * q)) - 1)
                assert got == want, (seed, q, n, k, xo, yo, oo)
                cases += 1
    print("ok", cases)


if __name__ == "__main__":
    main()

"""Child of test_gpu_peer_gather: world_size ranks on the local GPU(s) (gloo
for the IPC handle exchange and barriers), distributed_extract(gather="peer"):
every rank's kernels store their block range straight into rank 0's buffer."""
import os
import pathlib
import random
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from oracle import coracle
from paper_2402_14607_b200 import sharding


def main():
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ndev)
    torch.cuda.set_device(dev)
    rnd = random.Random(5)
    ok = 0
    for q, n, k, off in [(4, 64, 5000, 0), (56, 48, 700, 3), (13, 7, 1025, 5), (128, 8, 200, 0),
                         (16, 64, 4096, 0), (7, 5, 65, 1), (80, 71, 3, 2)]:
        nb = (off + k * q * n + 7) // 8
        xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
        got = sharding.distributed_extract(xb, yb, q, n, k, x_bit0=off, y_bit0=off,
                                           device=dev, gather="peer")
        if rank == 0:
            want = coracle.extract_eq(xb, yb, q, n, k, x_bit0=off, y_bit0=off)
            assert got == want, (q, n, k, off)
            ok += 1
        else:
            assert got is None
        # device-resident variant
        t = sharding.distributed_extract(xb, yb, q, n, k, x_bit0=off, y_bit0=off, device=dev,
                                         gather="peer", to_host=False)
        if rank == 0:
            assert t.is_cuda and t.cpu().numpy().tobytes() == want
    dist.destroy_process_group()
    if rank == 0:
        print("ok", ok)


if __name__ == "__main__":
    main()

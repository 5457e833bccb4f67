"""World-size-2 gloo run of the multi-process sharder on CPU.

Each rank computes its contiguous 64-aligned block range and rank 0 assembles
the output; the per-rank compute is the CPU oracle standing in for the device
(test-only), so this checks ranges, offsets and assembly, not the kernel (the
kernel's sharded output is checked on the GPU in test_gpu_parity)."""
import os
import random
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_compute(xv, yv, q, n, count, *, x_bit0=0, y_bit0=0):
    from oracle import coracle
    return coracle.extract_eq(bytes(xv), bytes(yv), q, n, count, x_bit0=x_bit0, y_bit0=y_bit0)


def _worker(rank, world, port, cases, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_14607_b200 import sharding
    try:
        for i, (xb, yb, q, n, k, off) in enumerate(cases):
            out = sharding.distributed_extract(xb, yb, q, n, k, x_bit0=off, y_bit0=off,
                                               compute=_oracle_compute)
            if rank == 0:
                results[i] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_sharded_extraction_matches_single(world):
    from oracle import coracle
    rnd = random.Random(77)
    cases = []
    for q, n, k in [(4, 64, 1000), (56, 48, 129), (13, 7, 257), (128, 8, 64), (80, 71, 3)]:
        off = rnd.randint(0, 7)
        nb = (off + k * q * n + 7) // 8
        cases.append((rnd.randbytes(nb), rnd.randbytes(nb), q, n, k, off))
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, cases, results), nprocs=world, join=True)
    for i, (xb, yb, q, n, k, off) in enumerate(cases):
        want = coracle.extract_eq(xb, yb, q, n, k, x_bit0=off, y_bit0=off)
        assert results[i] == want, (q, n, k)

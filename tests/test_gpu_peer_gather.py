"""distributed_extract(gather="peer"): output ranges stored by each rank's
kernels directly into rank 0's HBM buffer (CUDA IPC; NVLink peer stores on a
multi-GPU node).  Runs 2 ranks on whatever GPUs are visible -- on a one-GPU
box both ranks share the device, which exercises the IPC mapping and the range
logic (not peer bandwidth); no kernel waits on another rank's kernel."""
import pathlib
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

CHILD = pathlib.Path(__file__).with_name("gpu_peer_child.py")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_gather_two_ranks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    port = str(_port())
    procs = [subprocess.Popen([sys.executable, str(CHILD), str(r), "2", port],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    assert outs[0][0].startswith("ok 7"), outs[0]
